// cmg_kernels.cuh -- sm_100a kernels of the multigrid curvature V-cycle.
//
//   k_sweep_tpp   one colour of one level, one THREAD per patch (levels 1-3)
//                 == driver.sweep_layer colour step (driver.py:242-251) +
//                    color_corrections (driver.py:175-222)
//   k_sweep_bpp   one colour of one level, one CTA per patch (levels 4-6)
//   k_energy      level-1 curvature + fidelity + rel_u/PSNR partial sums
//                 (tangent.py:313-341, driver.py:161-166, :284-291)
//   k_finalize    per-image deterministic reduction, trace record and the
//                 stopping rule on device (driver.py:296-310)
//   k_pad_*       numpy-exact odd-reflection materialisation for images too
//                 small for single-chunk reflection (tangent.py:262-269)
//
// Semantics: all same-colour patches of one colour update u IN PLACE.  This is
// bit-identical to the reference's per-colour snapshot because a patch only
// reads its own pixels, its 1-pixel ring (other colours) and reflections of
// those; the general path reads a padded snapshot instead.
#pragma once

#include "cmg_device.cuh"

namespace cmg {

enum { MODE_MEAN = 0, MODE_GAUSS = 1 };
enum { PREC_EXACT = 0, PREC_FAST = 1 };
enum { SRC_INPLACE = 0, SRC_PADDED = 1 };

enum {
    ST_RUNNING = -1,
    ST_CONVERGED = 0,
    ST_NOT_CONVERGED = 2,
    ST_DIVERGED = 3,
    ST_NONFINITE = 5,
};

struct SolveParams {
    double alpha, half_alpha, eps, peak;
    int max_outer, inner, stop_rule, has_ref;
    long long npix;
    double w[7][16];    // backward-step weights per level (fbs.py:84-90)
    double den[7][16];  // 2 + w
};

// backward-step constants of one level, passed BY VALUE in the kernel
// arguments (constant bank) so the patch solve needs no dependent global load
struct BackK {
    int inner;
    double w0, den0, inv0;
};

struct ImgState {
    double F;         // last energy
    int cycle;        // index of last trace record
    int done;         // 1 once stopped
    int status;       // ST_*
    int bad;          // non-finite correction seen during the current cycle
    unsigned long long t0;
    // energy-fused cycle (the level-1 kernel of cycle g+1 computes and finalizes
    // the energy of u_g): started = the initial record exists; bad1 = non-finite
    // correction in the level-1 sweep now running, bad1_prev = in the previous
    // cycle's level-1 sweep (its later levels report through `bad`)
    int started;
    int bad1;
    int bad1_prev;
    int final_buf;  // rotation buffer holding the image's final u once it stopped (k_collect)
};

template <typename T>
struct SweepArgs {
    T* u;
    const T* f;
    long long istride;  // elements per image
    const T* upad;      // padded snapshot (SRC_PADDED)
    const T* fpad;
    long long pstride;
    int W;
    int m, n;
    int layer, s, r;
    int p, q, hc, wc;
    int flat, single;
    const SolveParams* P;
    ImgState* st;
    int dbg;  // diagnostics: bit0 skip planes, bit1 skip f*, bit2 skip apply, bit3 exit early
    BackK bk;
    // fast mean mode: per-patch sums of the padded f of this level ([B][mj][nj], fp64, computed once
    // per solve by k_patch_fsum), so f* = (sum f - sum u) / S^2 needs no f pixels; nullptr: unused
    const double* fsum;
    long long fs_img;
    int fs_ld;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Rare orderings, kept out of line so the hot kernels stay small (I-cache):
// f* of a colour class with a single patch column (NumPy coalesces the patch
// into one flat pairwise sum) ...
template <typename T, int S, class Acc, class AccF = Acc>
__device__ __noinline__ T fstar_flat_sum(const Acc U, const AccF F, int R0, int C0) {
    using O = X<T>;
    return O::add(T(0), pairwise_small<T>(S * S, [&](int e) {
        return O::sub(F(R0 + e / S, C0 + e % S), U(R0 + e / S, C0 + e % S));
    }));
}
// ... and the plane mean of a colour class holding a single patch
// (d.mean(axis=0) on a (iota,1,1) array is pairwise, not sequential).
template <typename T>
__device__ __noinline__ T pairwise_of(const T* v, int n) {
    return pairwise_any<T>(n, [&](int i) { return v[i]; });
}

// backward steps (driver.py:212-214, fbs.py:84-90): c_0 = 0, so the common
// single step is (c_half + w f*) / (2 + w); constants come from the kernel
// arguments (SweepArgs::bk), further steps from SolveParams
template <typename T, int LAYER, int PREC>
__device__ __forceinline__ T backward_steps(T chalf, T fstar, const SweepArgs<T>& a) {
    using O = X<T>;
    if (a.bk.inner == 1) {
        if constexpr (PREC == PREC_FAST)
            return (chalf + T(a.bk.w0) * fstar) * T(a.bk.inv0);
        else  // keep the reference's (0 + c_half) so even the sign of zero matches
            return O::div(O::add(O::add(T(0), chalf), O::mul(T(a.bk.w0), fstar)), T(a.bk.den0));
    }
    T c = T(0);
    const int lay = LAYER > 0 ? LAYER : a.layer;
    for (int t = 0; t < a.bk.inner; ++t)
        c = O::div(O::add(O::add(c, chalf), O::mul(T(a.P->w[lay][t]), fstar)), T(a.P->den[lay][t]));
    return c;
}

// ---------------------------------------------------------------------------
// Local solve of one patch (levels 1..3, compile-time plane tables).
// ---------------------------------------------------------------------------
template <typename T, int LAYER, int MODE, int PREC, class Acc>
__device__ __forceinline__ T patch_solve_ct(const Acc& U, const Acc& F, int R0, int C0, const SweepArgs<T>& a) {
    using O = X<T>;
    constexpr int S = (1 << LAYER) - 1;
    constexpr int R = 1 << (LAYER - 1);
    constexpr int NPL = 1 << (LAYER + 2);
    const int ci = R0 + R - 1, cc = C0 + R - 1;

    // f* = mean over the padded patch of (f - u)   (driver.py:244-246)
    T fstar;
    if constexpr (S == 1) {
        fstar = O::sub(F(R0, C0), U(R0, C0));
    } else {
        auto D = [&](int aa, int bb) { return O::sub(F(R0 + aa, C0 + bb), U(R0 + aa, C0 + bb)); };
        T acc;
        if (a.flat) {
            acc = fstar_flat_sum<T, S>(U, F, R0, C0);
        } else {
            acc = T(0);
#pragma unroll
            for (int aa = 0; aa < S; ++aa) acc = O::add(acc, pairwise_small<T>(S, [&](int bb) { return D(aa, bb); }));
        }
        fstar = O::div(acc, T(S * S));
    }

    const T uo = U(ci, cc);
    T chalf;
    if constexpr (MODE == MODE_MEAN) {
        if constexpr (PREC == PREC_FAST) {
            T sum = T(0);
            static_for<0, NPL / 2>([&](auto k) { sum += pair_fast<T, decltype(k)::value>(U, ci, cc, uo); });
            chalf = sum * T(1.0 / NPL);
        } else {
            T d[NPL];
            static_for<0, NPL>([&](auto l) { plane_exact<T, decltype(l)::value>(U, ci, cc, uo, &d[decltype(l)::value], nullptr); });
            T sum;
            if (a.single) {
                T tmp[NPL];
#pragma unroll
                for (int l = 0; l < NPL; ++l) tmp[l] = d[l];
                sum = pairwise_of<T>(tmp, NPL);
            } else {
                sum = d[0];
#pragma unroll
                for (int l = 1; l < NPL; ++l) sum = O::add(sum, d[l]);
            }
            chalf = div_pow2<T, NPL>(sum);  // NPL = 2^(J+2)
        }
    } else {
        T v[NPL];
        static_for<0, NPL>([&](auto l) { plane_exact<T, decltype(l)::value>(U, ci, cc, uo, nullptr, &v[decltype(l)::value]); });
        // np.argmin / np.argmax along planes: first index, first NaN wins
        int imin = 0, imax = 0;
        bool nanseen = isnan(v[0]);
#pragma unroll
        for (int l = 1; l < NPL; ++l) {
            if (!nanseen) {
                if (isnan(v[l])) {
                    nanseen = true;
                    imin = l;
                    imax = l;
                } else {
                    if (v[l] < v[imin]) imin = l;
                    if (v[l] > v[imax]) imax = l;
                }
            }
        }
        T vmin = v[0], vmax = v[0];
#pragma unroll
        for (int l = 1; l < NPL; ++l) {
            if (l == imin) vmin = v[l];
            if (l == imax) vmax = v[l];
        }
        const int star = (fabs(vmin) <= fabs(vmax)) ? imin : imax;
        plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::get(star), &chalf, nullptr);
    }

    return backward_steps<T, LAYER, PREC>(chalf, fstar, a);
}

template <typename T>
__device__ __forceinline__ void apply_patch(T* u, int m, int n, int R0, int C0, int S, T c) {
    const int r1 = min(R0 + S, m), c1 = min(C0 + S, n);
    for (int i = R0; i < r1; ++i)
        for (int k = C0; k < c1; ++k) {
            T* p = u + (long long)i * n + k;
            *p = X<T>::add(*p, c);
        }
}

// Border patches (odd reflection) take an out-of-line copy of the solve.
template <typename T, int LAYER, int MODE, int PREC>
__device__ __forceinline__ T patch_solve_ct_border(const T* u, const T* f, int R0, int C0, const SweepArgs<T>& a) {
    Reflect<T> U{u, a.m, a.n}, F{f, a.m, a.n};
    return patch_solve_ct<T, LAYER, MODE, PREC>(U, F, R0, C0, a);
}

template <typename T, int LAYER, int MODE, int PREC, int SRC>
__global__ void __launch_bounds__(256) k_sweep_tpp(SweepArgs<T> a) {
    pdl_sync();
    const int b = blockIdx.z;
    if (a.st[b].done) return;
    const int pc = blockIdx.x * blockDim.x + threadIdx.x;
    const int pr = blockIdx.y * blockDim.y + threadIdx.y;
    if (pc >= a.wc || pr >= a.hc) return;
    constexpr int S = (1 << LAYER) - 1;
    const int R0 = (2 * pr + a.p) * S, C0 = (2 * pc + a.q) * S;
    T* u = a.u + (long long)b * a.istride;
    const T* f = a.f + (long long)b * a.istride;
    T c;
    if constexpr (SRC == SRC_PADDED) {
        Padded<T> U{a.upad + (long long)b * a.pstride, a.W}, F{a.fpad + (long long)b * a.pstride, a.W};
        c = patch_solve_ct<T, LAYER, MODE, PREC>(U, F, R0, C0, a);
    } else {
        const bool inside = (R0 >= 1) && (C0 >= 1) && (R0 + S < a.m) && (C0 + S < a.n);
        if (inside) {
            Direct<T> U{u, a.n}, F{f, a.n};
            c = patch_solve_ct<T, LAYER, MODE, PREC>(U, F, R0, C0, a);
        } else {
            c = patch_solve_ct_border<T, LAYER, MODE, PREC>(u, f, R0, C0, a);
        }
    }
    if (!isfinite(c)) a.st[b].bad = 1;
    apply_patch(u, a.m, a.n, R0, C0, S, c);
}


// ---------------------------------------------------------------------------
// Team-per-patch sweep (levels 2-3): TS consecutive lanes of a warp cooperate
// on one patch -- rows of f* in parallel, planes split across lanes, the
// NumPy-ordered reductions replayed through warp shuffles.
// ---------------------------------------------------------------------------
template <typename T>
struct ArgBest {
    T v;
    int i;
    bool nan;
};

// np.argmin / np.argmax order: any NaN beats numbers (first NaN index wins),
// otherwise strictly better value, ties -> smaller index.
template <bool MIN, typename T>
__device__ __forceinline__ ArgBest<T> arg_better(const ArgBest<T>& a, const ArgBest<T>& b) {
    if (a.nan || b.nan) {
        if (a.nan && b.nan) return a.i <= b.i ? a : b;
        return a.nan ? a : b;
    }
    if (MIN ? (a.v < b.v) : (a.v > b.v)) return a;
    if (MIN ? (b.v < a.v) : (b.v > a.v)) return b;
    return a.i <= b.i ? a : b;
}

template <bool MIN, int TS, typename T>
__device__ __forceinline__ ArgBest<T> arg_reduce(ArgBest<T> x) {
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) {
        ArgBest<T> y;
        y.v = __shfl_xor_sync(0xffffffffu, x.v, o, TS);
        y.i = __shfl_xor_sync(0xffffffffu, x.i, o, TS);
        y.nan = __shfl_xor_sync(0xffffffffu, (int)x.nan, o, TS) != 0;
        x = arg_better<MIN>(x, y);
    }
    return x;
}

// fast mean mode: closed-form c_half of a patch, planes split
// over the TS lanes, then the backward steps
template <typename T, int LAYER, int TS, class Acc>
__device__ __forceinline__ T patch_chalf_fast_team(const Acc& U, int ci, int cc, int lane, T fstar,
                                                   const SweepArgs<T>& a) {
    constexpr int NPL = 1 << (LAYER + 2);
    constexpr int NPAIR = NPL / 2;
    constexpr unsigned FULL = 0xffffffffu;
    const T uo = U(ci, cc);
    T part = T(0);
#pragma unroll
    for (int k = 0; k < (NPAIR + TS - 1) / TS; ++k) {
        const int pi = lane + k * TS;
        if (pi < NPAIR) {
            const PlaneRT pl = PlaneRT::getg(2 * pi);
            const int Lq = pl.x0 * pl.x0 + pl.x1 * pl.x1;
            const T up = U(ci + pl.x0, cc + pl.x1), um = U(ci - pl.x0, cc - pl.x1);
            const T uq = U(ci + pl.y0, cc + pl.y1), umq = U(ci - pl.y0, cc - pl.y1);
            const T sp = up + um;
            const T N = sp - T(2) * uo;
            const T Dd = up - um;
            const T base = Dd * Dd + T(4 * Lq);
            const T Sa = sp - T(2) * uq, Sb = sp - T(2) * umq;
            part += (sqrt(T(Lq)) * N) * (frsqrt(Sa * Sa + base) + frsqrt(Sb * Sb + base));
        }
    }
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o, TS);
    return backward_steps<T, LAYER, PREC_FAST>(part * T(1.0 / NPL), fstar, a);
}

template <typename T, int LAYER, int MODE, int PREC, int TS, class Acc, class AccF = Acc>
__device__ __forceinline__ T patch_solve_team(const Acc& U, const AccF& F, int R0, int C0, int lane,
                                              const SweepArgs<T>& a, const double* fsum_patch = nullptr) {
    using O = X<T>;
    constexpr int S = (1 << LAYER) - 1;
    constexpr int R = 1 << (LAYER - 1);
    constexpr int NPL = 1 << (LAYER + 2);
    constexpr unsigned FULL = 0xffffffffu;
    // teams narrower than a patch row only exist for the fast mean mode with
    // per-patch f sums (large-job row-parity kernel, one thread per patch)
    static_assert(TS <= 32 && (32 % TS) == 0, "team size");
    static_assert(TS >= S || (MODE == MODE_MEAN && PREC == PREC_FAST), "team narrower than a patch row");
    const int ci = R0 + R - 1, cc = C0 + R - 1;
    auto D = [&](int aa, int bb) { return O::sub(F(R0 + aa, C0 + bb), U(R0 + aa, C0 + bb)); };

    if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        if (TS < S || fsum_patch) {  // f* = (sum f - sum u) / S^2 with the precomputed sum of f (fast mode only)
            T ur = T(0);
#pragma unroll
            for (int r = lane; r < S; r += TS) {
#pragma unroll
                for (int bb = 0; bb < S; ++bb) ur += U(R0 + r, C0 + bb);
            }
#pragma unroll
            for (int o = TS / 2; o > 0; o >>= 1) ur += __shfl_xor_sync(FULL, ur, o, TS);
            const T fstar = T((__ldg(fsum_patch) - (double)ur) * (1.0 / (S * S)));
            if constexpr (TS == 1) {  // one thread per patch: compile-time plane offsets
                const T uo = U(ci, cc);
                T sum = T(0);
                static_for<0, NPL / 2>([&](auto k) { sum += pair_fast<T, decltype(k)::value>(U, ci, cc, uo); });
                return backward_steps<T, LAYER, PREC_FAST>(sum * T(1.0 / NPL), fstar, a);
            }
            return patch_chalf_fast_team<T, LAYER, TS>(U, ci, cc, lane, fstar, a);
        }
    }
    if constexpr (TS < S) {
        return T(0);  // unreachable: TS < S implies the f-sum branch above
    } else {

    // f*: lane t owns row t (driver.py:244-246; rows sequential, each pairwise)
    T rowsum = T(0);
    if (a.dbg & 2) {
    } else if (a.flat) {
        if (lane == 0) rowsum = fstar_flat_sum<T, S>(U, F, R0, C0);
    } else if (lane < S) {
        rowsum = pairwise_small<T>(S, [&](int bb) { return D(lane, bb); });
    }
    T acc;
    if (a.flat) {
        acc = __shfl_sync(FULL, rowsum, 0, TS);
    } else {
        acc = T(0);
#pragma unroll
        for (int aa = 0; aa < S; ++aa) acc = O::add(acc, __shfl_sync(FULL, rowsum, aa, TS));
    }
    const T fstar = O::div(acc, T(S * S));

    const T uo = U(ci, cc);
    T chalf;
    if (a.dbg & 1) {
        chalf = uo;
    } else if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        constexpr int NPAIR = NPL / 2;
        T part = T(0);
#pragma unroll
        for (int k = 0; k < (NPAIR + TS - 1) / TS; ++k) {
            const int pi = lane + k * TS;
            if (pi < NPAIR) {
                const PlaneRT pl = PlaneRT::getg(2 * pi);
                const int Lq = pl.x0 * pl.x0 + pl.x1 * pl.x1;
                const T up = U(ci + pl.x0, cc + pl.x1), um = U(ci - pl.x0, cc - pl.x1);
                const T uq = U(ci + pl.y0, cc + pl.y1), umq = U(ci - pl.y0, cc - pl.y1);
                const T sp = up + um;
                const T N = sp - T(2) * uo;
                const T Dd = up - um;
                const T base = Dd * Dd + T(4 * Lq);
                const T Sa = sp - T(2) * uq, Sb = sp - T(2) * umq;
                part += (sqrt(T(Lq)) * N) * (frsqrt(Sa * Sa + base) + frsqrt(Sb * Sb + base));
            }
        }
#pragma unroll
        for (int o = TS / 2; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o, TS);
        chalf = part * T(1.0 / NPL);
    } else if constexpr (MODE == MODE_MEAN) {
        constexpr int PPL = NPL / TS;
        T d[PPL];
#pragma unroll
        for (int k = 0; k < PPL; ++k) plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::getg(lane + k * TS), &d[k], nullptr);
        T sum;
        if (a.single) {
            T all[NPL];
#pragma unroll
            for (int l = 0; l < NPL; ++l) all[l] = __shfl_sync(FULL, d[l / TS], l % TS, TS);
            sum = pairwise_of<T>(all, NPL);
        } else {
            sum = __shfl_sync(FULL, d[0], 0, TS);
#pragma unroll
            for (int l = 1; l < NPL; ++l) sum = O::add(sum, __shfl_sync(FULL, d[l / TS], l % TS, TS));
        }
        chalf = div_pow2<T, NPL>(sum);  // NPL = 2^(J+2)
    } else {
        constexpr int PPL = NPL / TS;
        ArgBest<T> bmin, bmax;
#pragma unroll
        for (int k = 0; k < PPL; ++k) {
            T v;
            plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::getg(lane + k * TS), nullptr, &v);
            ArgBest<T> c{v, lane + k * TS, (bool)isnan(v)};
            if (k == 0) {
                bmin = c;
                bmax = c;
            } else {
                bmin = arg_better<true>(bmin, c);
                bmax = arg_better<false>(bmax, c);
            }
        }
        bmin = arg_reduce<true, TS>(bmin);
        bmax = arg_reduce<false, TS>(bmax);
        const int star = (fabs(bmin.v) <= fabs(bmax.v)) ? bmin.i : bmax.i;
        T ph = T(0);
        if (lane == 0) plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::getg(star), &ph, nullptr);
        chalf = __shfl_sync(FULL, ph, 0, TS);
    }
    return backward_steps<T, LAYER, PREC>(chalf, fstar, a);
    }
}

template <typename T, int LAYER, int MODE, int PREC, int TS>
__device__ __forceinline__ T patch_solve_team_border(const T* u, const T* f, int R0, int C0, int lane,
                                                  const SweepArgs<T>& a, const double* fsp = nullptr) {
    Reflect<T> U{u, a.m, a.n}, F{f, a.m, a.n};
    return patch_solve_team<T, LAYER, MODE, PREC, TS>(U, F, R0, C0, lane, a, fsp);
}

template <typename T, int LAYER, int MODE, int PREC, int SRC, int TS>
__global__ void __launch_bounds__(256) k_sweep_team(SweepArgs<T> a) {
    pdl_sync();
    const int b = blockIdx.z;
    if (a.st[b].done) return;  // uniform per block
    constexpr int S = (1 << LAYER) - 1;
    const int lane = threadIdx.x % TS;
    const int npatch = a.hc * a.wc;  // < 2^31 (m*n < 2^31)
    int idx = (int)blockIdx.x * (256 / TS) + (int)threadIdx.x / TS;
    const bool valid = idx < npatch;
    if (!valid) idx = npatch - 1;  // keep the whole warp converged for the shuffles
    const int pr = idx / a.wc, pc = idx - pr * a.wc;
    const int R0 = (2 * pr + a.p) * S, C0 = (2 * pc + a.q) * S;
    T* u = a.u + (long long)b * a.istride;
    const T* f = a.f + (long long)b * a.istride;
    if (a.dbg & 8) return;
    T c;
    if constexpr (SRC == SRC_PADDED) {
        Padded<T> U{a.upad + (long long)b * a.pstride, a.W}, F{a.fpad + (long long)b * a.pstride, a.W};
        c = patch_solve_team<T, LAYER, MODE, PREC, TS>(U, F, R0, C0, lane, a);
    } else {
        const double* fsp =
            a.fsum ? a.fsum + (long long)b * a.fs_img + (long long)(R0 / S) * a.fs_ld + C0 / S : nullptr;
        const bool inside = (R0 >= 1) && (C0 >= 1) && (R0 + S < a.m) && (C0 + S < a.n);
        if (__all_sync(0xffffffffu, inside)) {
            Direct<T> U{u, a.n}, F{f, a.n};
            c = patch_solve_team<T, LAYER, MODE, PREC, TS>(U, F, R0, C0, lane, a, fsp);
        } else {
            c = patch_solve_team_border<T, LAYER, MODE, PREC, TS>(u, f, R0, C0, lane, a, fsp);
        }
    }
    if (!valid || (a.dbg & 4)) return;
    if (lane == 0 && !isfinite(c)) a.st[b].bad = 1;
    // prolongation (hierarchy.py:117-126): the lane's loads are all issued before its
    // first store (the plain read-modify-write loop made one round trip per element)
    constexpr int NIT = (S * S + TS - 1) / TS;
    T v[NIT];
#pragma unroll
    for (int t = 0; t < NIT; ++t) {
        const int e = lane + t * TS;
        const int i = R0 + e / S, k = C0 + e % S;
        if (e < S * S && i < a.m && k < a.n) v[t] = u[(long long)i * a.n + k];
    }
#pragma unroll
    for (int t = 0; t < NIT; ++t) {
        const int e = lane + t * TS;
        const int i = R0 + e / S, k = C0 + e % S;
        if (e < S * S && i < a.m && k < a.n) u[(long long)i * a.n + k] = X<T>::add(v[t], c);
    }
}

// ---------------------------------------------------------------------------
// One CTA per patch (coarse levels, runtime plane table).  Always the exact
// NumPy operation order.
// ---------------------------------------------------------------------------
template <typename T, int MODE, class Acc>
__device__ __forceinline__ void bpp_body(const Acc& U, const Acc& F, int R0, int C0, const SweepArgs<T>& a,
                                         T* sh_rows, T* sh_vals, T* sh_c, ArgBest<T>* sh_best) {
    using O = X<T>;
    const int S = a.s, NPL = 1 << (a.layer + 2);
    const int ci = R0 + a.r - 1, cc = C0 + a.r - 1;
    const int tid = threadIdx.x;
    auto D = [&](int aa, int bb) { return O::sub(F(R0 + aa, C0 + bb), U(R0 + aa, C0 + bb)); };
    if (a.flat) {
        if (tid == 0) sh_rows[0] = pairwise_any<T>(S * S, [&](int e) { return D(e / S, e % S); });
    } else {
        // row sums in numpy's pairwise order (8 <= S < 128: eight strided accumulators,
        // a fixed combination tree, then the remainder): eight lanes per row, lane t
        // owns accumulator t, so a row's loads are coalesced and short
        const int t = tid & 7, rg = tid >> 3, nrg = blockDim.x >> 3;
        const int n8 = S - (S % 8);
        for (int base = 0; base < S; base += nrg) {
            const bool act = base + rg < S;
            const int aa = act ? base + rg : S - 1;
            T r = D(aa, t);
            for (int i = 8; i < n8; i += 8) r = O::add(r, D(aa, i + t));
            r = O::add(r, __shfl_down_sync(0xffffffffu, r, 1, 8));  // t even: r_t + r_{t+1}
            r = O::add(r, __shfl_down_sync(0xffffffffu, r, 2, 8));  // t = 0, 4: pairs of pairs
            r = O::add(r, __shfl_down_sync(0xffffffffu, r, 4, 8));  // t = 0: the tree's root
            if (t == 0 && act) {
                for (int i = n8; i < S; ++i) r = O::add(r, D(aa, i));
                sh_rows[aa] = r;
            }
        }
    }
    const T uo = U(ci, cc);
    for (int l = tid; l < NPL; l += blockDim.x) {
        T v;
        // lane-divergent plane index: the packed global table (constant memory would serialise)
        if (MODE == MODE_MEAN)
            plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::getg(l), &v, nullptr);
        else
            plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::getg(l), nullptr, &v);
        sh_vals[l] = v;
    }
    if (MODE != MODE_MEAN) {
        // Gaussian mode: lexicographic (value, index, NaN) reductions of the thread's
        // planes, then of the warp; thread 0 combines the warps
        // (a thread or warp without a plane holds +-inf with the largest index, which loses
        // against every plane: NaN beats it, any number is at least as good with a lower index)
        ArgBest<T> bmin{T(INFINITY), 0x7fffffff, false}, bmax{T(-INFINITY), 0x7fffffff, false};
        for (int l = tid; l < NPL; l += blockDim.x) {
            const T v = sh_vals[l];  // this thread's own value
            const ArgBest<T> c{v, l, (bool)isnan(v)};
            bmin = arg_better<true>(bmin, c);
            bmax = arg_better<false>(bmax, c);
        }
        bmin = arg_reduce<true, 32>(bmin);
        bmax = arg_reduce<false, 32>(bmax);
        if ((tid & 31) == 0) {
            sh_best[2 * (tid >> 5)] = bmin;
            sh_best[2 * (tid >> 5) + 1] = bmax;
        }
    }
    __syncthreads();
    if (tid == 0) {
        T acc;
        if (a.flat) {
            acc = O::add(T(0), sh_rows[0]);
        } else {
            acc = T(0);
#pragma unroll 8
            for (int aa = 0; aa < S; ++aa) acc = O::add(acc, sh_rows[aa]);
        }
        const T fstar = O::div(acc, T(S * S));
        T chalf;
        if (MODE == MODE_MEAN) {
            T sum;
            if (a.single) {
                sum = pairwise_any<T>(NPL, [&](int i) { return sh_vals[i]; });
            } else {
                sum = sh_vals[0];
#pragma unroll 8
                for (int l = 1; l < NPL; ++l) sum = O::add(sum, sh_vals[l]);
            }
            chalf = O::mul(sum, T(1.0 / NPL));  // NPL = 2^(J+2): exact reciprocal, same as the division
        } else {
            // np.argmin / np.argmax from the per-warp results (first NaN wins, ties -> lower index)
            ArgBest<T> bmin = sh_best[0], bmax = sh_best[1];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                bmin = arg_better<true>(bmin, sh_best[2 * w]);
                bmax = arg_better<false>(bmax, sh_best[2 * w + 1]);
            }
            const int star = (fabs(bmin.v) <= fabs(bmax.v)) ? bmin.i : bmax.i;
            plane_exact_rt<T>(U, ci, cc, uo, PlaneRT::get(star), &chalf, nullptr);
        }
        T c = T(0);
        for (int t = 0; t < a.P->inner; ++t)
            c = O::div(O::add(O::add(c, chalf), O::mul(T(a.P->w[a.layer][t]), fstar)), T(a.P->den[a.layer][t]));
        *sh_c = c;
    }
}

template <typename T, int MODE, int SRC>
__global__ void __launch_bounds__(256) k_sweep_bpp(SweepArgs<T> a) {
    pdl_sync();
    __shared__ T sh_rows[64];
    __shared__ T sh_vals[256];
    __shared__ T sh_c;
    __shared__ ArgBest<T> sh_best[16];  // per-warp argmin / argmax (Gaussian mode, <= 8 warps)
    const int b = blockIdx.z;
    if (a.st[b].done) return;
    const int pc = blockIdx.x, pr = blockIdx.y;
    const int S = a.s;
    const int R0 = (2 * pr + a.p) * S, C0 = (2 * pc + a.q) * S;
    T* u = a.u + (long long)b * a.istride;
    const T* f = a.f + (long long)b * a.istride;
    if constexpr (SRC == SRC_PADDED) {
        Padded<T> U{a.upad + (long long)b * a.pstride, a.W}, F{a.fpad + (long long)b * a.pstride, a.W};
        bpp_body<T, MODE>(U, F, R0, C0, a, sh_rows, sh_vals, &sh_c, sh_best);
    } else {
        const bool inside = (R0 >= 1) && (C0 >= 1) && (R0 + S < a.m) && (C0 + S < a.n);
        if (inside) {
            Direct<T> U{u, a.n}, F{f, a.n};
            bpp_body<T, MODE>(U, F, R0, C0, a, sh_rows, sh_vals, &sh_c, sh_best);
        } else {
            Reflect<T> U{u, a.m, a.n}, F{f, a.m, a.n};
            bpp_body<T, MODE>(U, F, R0, C0, a, sh_rows, sh_vals, &sh_c, sh_best);
        }
    }
    __syncthreads();
    const T c = sh_c;
    if (threadIdx.x == 0 && !isfinite(c)) a.st[b].bad = 1;
    const int r1 = min(R0 + S, a.m), c1 = min(C0 + S, a.n);
    const int w = c1 - C0, h = r1 - R0;
    // prolongation u += c (hierarchy.py:117-126): a thread per column (w <= 63) and
    // row lane, eight rows' loads in flight before the first store (the plain
    // read-modify-write loop made one memory round trip per element)
    const int col = threadIdx.x & 63, rl = threadIdx.x >> 6, nrl = blockDim.x >> 6;
    if (col < w) {
        T* base = u + (long long)R0 * a.n + C0 + col;
        for (int r = rl; r < h; r += 8 * nrl) {
            T v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (r + j * nrl < h) v[j] = base[(long long)(r + j * nrl) * a.n];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (r + j * nrl < h) base[(long long)(r + j * nrl) * a.n] = X<T>::add(v[j], c);
        }
    }
}

// ---------------------------------------------------------------------------
// Energy: per-pixel level-1 curvature (closed form kappa_p = N_p / (2|p|^2),
// SURVEY App. B; equal to tangent.curvature_field up to rounding) and the
// fidelity / rel_u / PSNR sums, accumulated in fp64.
// ---------------------------------------------------------------------------
struct EnergyArgs {
    const void* u;
    const void* f;
    const void* uprev;
    const void* ref;
    const void* upad;  // padded (pad 1) snapshot when SRC_PADDED
    long long istride, pstride;
    int m, n, W, mode, nbx;
    int ncb;               // k_energy: column chunks per row band (nbx = row bands * ncb)
    long long e_lo, e_hi;  // pixel index range of the sums (whole image: 0..m*n)
    double* partials;      // [B][nbx][5]
    const ImgState* st;
};

constexpr int NSUM = 5;  // curv, fid, |du|, |u|, (u-ref)^2

// level-1 curvature term of one pixel from its 3x3 neighbourhood, in the
// accumulation precision A (double for fp64 images, float for fp32 images;
// the sums are accumulated in double either way).  kappa_p = (u+p + u-p -
// 2 u) / (2 |p|^2) is evaluated as fma(u+p + u-p, 1/(2|p|^2), -u/|p|^2):
// the scalings are powers of two, so this is the same correctly rounded value
// with one instruction less.  A NaN anywhere makes the term NaN (np.min /
// np.max propagate NaN); for fp32 the NaN-propagating min/max instructions do
// that, for fp64 an explicit test.
__device__ __forceinline__ float fmin_nan(float a, float b) {
    float d;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

template <typename A>
__device__ __forceinline__ A curv_term(A uo, A uE, A uW, A uN, A uS, A uNE, A uSW, A uNW, A uSE, int mode) {
    const A h = A(-0.5) * uo;
    const A k0 = fma(uE + uW, A(0.5), -uo);
    const A k1 = fma(uN + uS, A(0.5), -uo);
    const A k2 = fma(uNE + uSW, A(0.25), h);
    const A k3 = fma(uNW + uSE, A(0.25), h);
    if constexpr (sizeof(A) == 4) {
        const float kmin = fmin_nan(fmin_nan(k0, k1), fmin_nan(k2, k3));
        const float kmax = fmax_nan(fmax_nan(k0, k1), fmax_nan(k2, k3));
        return (mode == MODE_MEAN) ? fabsf(0.5f * (kmin + kmax)) : fabsf(kmin * kmax);
    } else {
        const A kmin = fmin(fmin(k0, k1), fmin(k2, k3));
        const A kmax = fmax(fmax(k0, k1), fmax(k2, k3));
        A term = (mode == MODE_MEAN) ? fabs(A(0.5) * (kmin + kmax)) : fabs(kmin * kmax);
        if (isnan(k0) || isnan(k1) || isnan(k2) || isnan(k3)) term = A(NAN);
        return term;
    }
}

struct TraceArgs {
    double* energy;  // [B][cap]
    double* rel_e;
    double* rel_u;
    double* psnr;
    double* seconds;
    int cap;
    int* ndone;
    double* eonly;  // energy-only mode output [B] (nullptr in solve)
    double* raw5;   // raw partial sums [B][5] (strip mode), or nullptr
};

// Finalize one image (one CTA): reduce its partials in a fixed order, record
// the trace and apply the stopping rule (driver.py:294-310).  Returns true
// if the image is (now) done.
// initial: 1 = record cycle 0, 0 = record the next cycle, 2 = energy-fused
// cycle (record 0 if the image has not started, else the next cycle; the
// non-finite flag of the cycle is `bad` | `bad1_prev`).  `shf` is >= NSUM x 256
// doubles of shared scratch; the first min(256, block size) threads reduce.
static __device__ __noinline__ void finalize_image_s(int b, const double* partials, int nbx, const SolveParams* P,
                                              ImgState* st, TraceArgs tr, int initial, double (*shf)[256], int buf) {
    ImgState& S = st[b];
    const bool efused = initial == 2;
    if (efused) initial = S.started ? 0 : 1;
    if (!initial && tr.eonly == nullptr && tr.raw5 == nullptr && S.done) return;
    const int tid = threadIdx.x;
    const int nth = min((int)blockDim.x, 256);  // reducing threads (CTAs of fewer than 256 threads: 192)
    double acc[NSUM] = {0, 0, 0, 0, 0};
    if (tid < nth) {
#pragma unroll 4
        for (int i = tid; i < nbx; i += nth)
#pragma unroll
            for (int s = 0; s < NSUM; ++s) acc[s] += __ldcg(&partials[((long long)b * nbx + i) * NSUM + s]);
#pragma unroll
        for (int s = 0; s < NSUM; ++s) shf[s][tid] = acc[s];
    }
    for (int t = nth + tid; t < 256; t += blockDim.x)  // the tree below runs over 256 slots
#pragma unroll
        for (int s = 0; s < NSUM; ++s) shf[s][t] = 0.0;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (tid < w)
#pragma unroll
            for (int s = 0; s < NSUM; ++s) shf[s][tid] += shf[s][tid + w];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double curv = shf[0][0], fid = shf[1][0], du = shf[2][0], au = shf[3][0], dr = shf[4][0];
    if (tr.raw5) {
        for (int s = 0; s < NSUM; ++s) tr.raw5[b * NSUM + s] = shf[s][0];
        return;
    }
    const double F = curv + P->half_alpha * fid;
    if (tr.eonly) {
        tr.eonly[b] = F;
        return;
    }
    const unsigned long long now = globaltimer();
    double ps = __longlong_as_double(0x7ff8000000000000ULL);
    if (P->has_ref) {
        const double mse = dr / (double)P->npix;
        ps = (mse == 0.0) ? __longlong_as_double(0x7ff0000000000000ULL) : 10.0 * log10(P->peak * P->peak / mse);
    }
    const long long base = (long long)b * tr.cap;
    if (initial) {
        S.F = F;
        S.cycle = 0;
        S.done = 0;
        S.status = ST_RUNNING;
        S.bad = 0;
        S.started = 1;
        if (efused) {
            S.bad1_prev = S.bad1;
            S.bad1 = 0;
        }
        S.t0 = now;
        tr.energy[base] = F;
        tr.rel_e[base] = __longlong_as_double(0x7ff8000000000000ULL);
        tr.rel_u[base] = __longlong_as_double(0x7ff8000000000000ULL);
        tr.psnr[base] = ps;
        tr.seconds[base] = 0.0;
        return;
    }
    const int kk = S.cycle + 1;
    int badc = S.bad;
    if (efused) {
        badc |= S.bad1_prev;
        S.bad1_prev = S.bad1;
        S.bad1 = 0;
        S.bad = 0;
    }
    if (badc) {
        S.status = ST_NONFINITE;
        S.final_buf = buf;
        S.done = 1;
        atomicAdd(tr.ndone, 1);
        return;
    }
    if (!isfinite(F)) {
        tr.energy[base + kk] = F;
        S.status = ST_DIVERGED;
        S.final_buf = buf;
        S.done = 1;
        atomicAdd(tr.ndone, 1);
        return;
    }
    // rel_err_energy (driver.py:146-150), _rel_u_guarded (driver.py:161-166)
    const double re = (F == 0.0) ? fabs(S.F) : fabs(F - S.F) / fabs(F);
    const double ru = (au == 0.0) ? ((du == 0.0) ? 0.0 : __longlong_as_double(0x7ff0000000000000ULL)) : du / au;
    tr.energy[base + kk] = F;
    tr.rel_e[base + kk] = re;
    tr.rel_u[base + kk] = ru;
    tr.psnr[base + kk] = ps;
    tr.seconds[base + kk] = (double)(now - S.t0) * 1e-9;
    S.F = F;
    S.cycle = kk;
    const double crit = (P->stop_rule == 0) ? re : ru;
    if (crit <= P->eps) {
        S.status = ST_CONVERGED;
        S.final_buf = buf;
        S.done = 1;
        atomicAdd(tr.ndone, 1);
    } else if (kk >= P->max_outer) {
        S.status = ST_NOT_CONVERGED;
        S.final_buf = buf;
        S.done = 1;
        atomicAdd(tr.ndone, 1);
    }
}

__device__ __forceinline__ void finalize_image(int b, const double* partials, int nbx, const SolveParams* P,
                                               ImgState* st, const TraceArgs& tr, int initial, int buf = 0) {
    __shared__ double shf[NSUM][256];
    finalize_image_s(b, partials, nbx, P, st, tr, initial, shf, buf);
}

static __global__ void __launch_bounds__(256) k_finalize(const double* partials, int nbx, const SolveParams* P,
                                                         ImgState* st, TraceArgs tr, int initial, int buf) {
    pdl_sync();
    finalize_image(blockIdx.x, partials, nbx, P, st, tr, initial, buf);
}

// Energy + finalize in one launch: 32x8 pixel tiles (grid-stride), per-CTA
// fp64 partials, and the LAST CTA of each image (ticket counter) reduces
// them in a fixed order and runs finalize_image; the last image to finalize
// also sets the graph's WHILE condition.  Deterministic regardless of which
// CTA finishes last.
struct EnergyFin {
    TraceArgs tr;
    const SolveParams* P;
    ImgState* stw;
    int* tickets;     // [B] per-image CTA counters (self-resetting)
    int* img_ticket;  // [1] images finalized this cycle (self-resetting)
    int initial;
    unsigned long long cond;  // cudaGraphConditionalHandle (0: none)
    int B;
    int buf;  // rotation buffer index of the u being finalized (ImgState::final_buf)
};

// deterministic CTA reduction of the five sums -> partials[b][blockIdx.x];
// the last CTA of the image (ticket) finalizes it, and the last image sets
// the graph's WHILE condition
__device__ __forceinline__ void energy_reduce_finalize(const double (&acc)[NSUM], const EnergyArgs& a,
                                                       const EnergyFin& fz, int b) {
    const int tid = threadIdx.x;
    __shared__ double sh[NSUM][32];
    __shared__ int last;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int s = 0; s < NSUM; ++s) {
        double v = acc[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) sh[s][wid] = v;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
#pragma unroll
        for (int s = 0; s < NSUM; ++s) {
            double v = lane < nw ? sh[s][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) a.partials[((long long)b * a.nbx + blockIdx.x) * NSUM + s] = v;
        }
    }
    if (fz.tickets == nullptr) return;  // finalize launched separately
    __threadfence();
    if (tid == 0) last = (atomicAdd(&fz.tickets[b], 1) == a.nbx - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) fz.tickets[b] = 0;
    finalize_image(b, a.partials, a.nbx, fz.P, fz.stw, fz.tr, fz.initial, fz.buf);
    if (fz.cond == 0ULL || tid != 0) return;
    __threadfence();
    if (atomicAdd(fz.img_ticket, 1) == fz.B - 1) {
        *fz.img_ticket = 0;
        __threadfence();
        cudaGraphSetConditional((cudaGraphConditionalHandle)fz.cond, (*((volatile int*)fz.tr.ndone) < fz.B) ? 1u : 0u);
    }
}

// ---- energy fused into a level-1 tile kernel (energy-fused cycle) ----------
// (1) at the start, the CTA's fp64 sums of its owned pixels -> partials[b][cta]
__device__ __forceinline__ void cta_sums_store(const double (&acc)[NSUM], double* partials, int nbx, int cta,
                                               int b) {
    __shared__ double sh[NSUM][32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int s = 0; s < NSUM; ++s) {
        double v = acc[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) sh[s][wid] = v;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
#pragma unroll
        for (int s = 0; s < NSUM; ++s) {
            double v = lane < nw ? sh[s][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) partials[((long long)b * nbx + cta) * NSUM + s] = v;
        }
        // the writer fences here, long before its ticket (efused_ticket): the image's last
        // CTA then sees every CTA's sums without an all-thread fence behind the tile stores
        if (lane == 0) __threadfence();
    }
}

// (2) at the end (shared memory free), the ticket: the image's last CTA
// finalizes it (fixed-order reduction of the partials, trace, stopping rule)
// using `scratch` (>= NSUM x 256 doubles), and the last image sets the WHILE
// condition.  Every CTA of every image calls this, stopped images included.
__device__ __forceinline__ void efused_ticket(const EnergyFin& fz, const double* partials, int nbx, int b,
                                              double* scratch) {
    __shared__ int last;
    const int tid = threadIdx.x;
    // (thread 0 wrote and fenced this CTA's sums in cta_sums_store and fences its
    // non-finite flag where it sets it; the tile stores need no fence: nothing
    // before the next kernel reads them)
    __syncthreads();
    if (tid == 0) last = (atomicAdd(&fz.tickets[b], 1) == nbx - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0) fz.tickets[b] = 0;
    finalize_image_s(b, partials, nbx, fz.P, fz.stw, fz.tr, 2, reinterpret_cast<double (*)[256]>(scratch), fz.buf);
    if (fz.cond == 0ULL || tid != 0) return;
    __threadfence();
    if (atomicAdd(fz.img_ticket, 1) == fz.B - 1) {
        *fz.img_ticket = 0;
        __threadfence();
        cudaGraphSetConditional((cudaGraphConditionalHandle)fz.cond, (*((volatile int*)fz.tr.ndone) < fz.B) ? 1u : 0u);
    }
}

template <typename T, int SRC, int NT = 256>
__global__ void __launch_bounds__(NT, NT == 512 ? 2 : 1) k_energy(EnergyArgs a, EnergyFin fz) {
    pdl_sync();
    using A = T;
    const int b = blockIdx.y;
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    double acc[NSUM] = {0, 0, 0, 0, 0};
    if (!a.st[b].done) {
        const T* u = (const T*)a.u + (long long)b * a.istride;
        const T* f = (const T*)a.f + (long long)b * a.istride;
        const T* up = (const T*)a.uprev + (long long)b * a.istride;
        const T* rf = a.ref ? (const T*)a.ref + (long long)b * a.istride : nullptr;
        const int n = a.n, m = a.m;
        const int r_lo = (int)(a.e_lo / n), r_hi = (int)(a.e_hi / n);
        // each CTA owns a band of rows x a chunk of columns; a thread walks down
        // its columns keeping the 3x3 neighbourhood in registers (3 new u loads
        // per pixel).  Small images use many short bands (latency-bound pass).
        const int rows = r_hi - r_lo;
        const int nrb = a.nbx / a.ncb, rb = blockIdx.x / a.ncb, cb = blockIdx.x % a.ncb;
        const int band = (rows + nrb - 1) / nrb;
        const int i0 = r_lo + rb * band, i1 = min(r_hi, i0 + band);
        const int cw = (n + a.ncb - 1) / a.ncb;
        const int k1 = min(n, (cb + 1) * cw);
        for (int k = cb * cw + tid; k < k1 && i0 < i1; k += blockDim.x) {
            const bool kin = (k >= 1) && (k + 1 < n);
            auto ldrow = [&](int i, A& wv, A& cv, A& ev) {
                if (SRC == SRC_PADDED) {
                    Padded<T> U{(const T*)a.upad + (long long)b * a.pstride, a.W};
                    wv = (A)U(i, k - 1);
                    cv = (A)U(i, k);
                    ev = (A)U(i, k + 1);
                } else if (kin && i >= 0 && i < m) {
                    const T* r = u + (long long)i * n + k;
                    wv = (A)r[-1];
                    cv = (A)r[0];
                    ev = (A)r[1];
                } else {
                    Reflect<T> U{u, m, n};
                    wv = (A)U(i, k - 1);
                    cv = (A)U(i, k);
                    ev = (A)U(i, k + 1);
                }
            };
            A nw, nc, ne, cw, cc, ce, sw, sc, se;
            ldrow(i0 - 1, nw, nc, ne);
            ldrow(i0, cw, cc, ce);
            // per-pixel terms accumulate in fp64 (fp32 images: the curvature term is
            // evaluated in fp32, the other terms from exact fp64 differences)
            double loc[NSUM] = {0, 0, 0, 0, 0};
            int cnt = 0;
            for (int i = i0; i < i1; ++i) {
                ldrow(i + 1, sw, sc, se);
                const long long e = (long long)i * n + k;
                const double fv = (double)f[e], pv = (double)up[e], c64 = (double)cc;
                loc[0] += (double)curv_term<A>(cc, ce, cw, nc, sc, ne, sw, nw, se, a.mode);
                const double d = c64 - fv;
                loc[1] += d * d;
                loc[2] += fabs(c64 - pv);
                loc[3] += fabs(c64);
                if (rf) {
                    const double dr = c64 - (double)rf[e];
                    loc[4] += dr * dr;
                }
                if (++cnt == 8) {  // 8-row partial sums, then the band accumulators
#pragma unroll
                    for (int s = 0; s < NSUM; ++s) {
                        acc[s] += loc[s];
                        loc[s] = 0.0;
                    }
                    cnt = 0;
                }
                nw = cw; nc = cc; ne = ce;
                cw = sw; cc = sc; ce = se;
            }
#pragma unroll
            for (int s = 0; s < NSUM; ++s) acc[s] += loc[s];
        }
    }
    energy_reduce_finalize(acc, a, fz, b);
}

// After a solve: images whose final u is not in rotation buffer 0 (they
// stopped in another cycle of the graph body; later kernels skipped them)
template <typename T>
__global__ void k_collect(T* u0, const T* u1, const T* u2, long long N, const ImgState* st) {
    const int b = blockIdx.y;
    const int fb = st[b].final_buf;
    if (fb == 0) return;
    const T* src = (fb == 1 ? u1 : u2) + (long long)b * N;
    T* dst = u0 + (long long)b * N;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x)
        dst[e] = src[e];
}

// Per-patch sums of the odd-padded f of one level (fast mean mode: f* =
// (sum f - sum u) / S^2, f is constant through a solve).  One thread per group
// of four horizontally adjacent patches: inside the image a group's row is
// 4 S consecutive pixels, read as S 16-byte loads (fp32, rows a multiple of 4
// pixels long); every pixel is added to its patch's fp64 sum in row-major
// order, as the one-patch path (groups touching the padding) does.
template <typename T, int S>
__global__ void k_patch_fsum(const T* __restrict__ f, double* out, int m, int n, int mj, int nj, long long istride) {
    pdl_sync();
    const int b = blockIdx.y;
    const long long np = (long long)mj * nj;
    const int ng = (nj + 3) / 4;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)mj * ng) return;
    const int pr = (int)(e / ng), pc0 = 4 * (int)(e % ng);
    const T* fb = f + (long long)b * istride;
    double* ob = out + (long long)b * np + (long long)pr * nj + pc0;
    if constexpr (sizeof(T) == 4) {
        if ((n & 3) == 0 && pr * S + S <= m && (pc0 + 4) * S <= n) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const float4* row = reinterpret_cast<const float4*>(fb + (long long)pr * S * n + (long long)pc0 * S);
#pragma unroll
            for (int i = 0; i < S; ++i) {
                float v[4 * S];
#pragma unroll
                for (int q = 0; q < S; ++q) {
                    const float4 w = __ldg(row + (long long)i * (n / 4) + q);
                    v[4 * q] = w.x;
                    v[4 * q + 1] = w.y;
                    v[4 * q + 2] = w.z;
                    v[4 * q + 3] = w.w;
                }
#pragma unroll
                for (int pp = 0; pp < 4; ++pp)
#pragma unroll
                    for (int k = 0; k < S; ++k) acc[pp] += (double)v[pp * S + k];
            }
#pragma unroll
            for (int pp = 0; pp < 4; ++pp) ob[pp] = acc[pp];
            return;
        }
    }
    const Reflect<T> F{fb, m, n};
    for (int pp = 0; pp < 4 && pc0 + pp < nj; ++pp) {
        double acc = 0.0;
        for (int i = 0; i < S; ++i)
            for (int k = 0; k < S; ++k) acc += (double)F(pr * S + i, (pc0 + pp) * S + k);
        ob[pp] = acc;
    }
}

// ---------------------------------------------------------------------------
// numpy-exact odd reflection materialisation (np.pad reflect/odd, including
// iterated chunks and the singleton 'edge' case; numpy _set_reflect_both).
// ---------------------------------------------------------------------------
template <typename T>
__device__ void reflect_line(T* line, long long stride, int left, int len, int right) {
    if (len == 1) {
        const T e = line[(long long)left * stride];
        for (int i = 0; i < left; ++i) line[(long long)i * stride] = e;
        for (int i = 0; i < right; ++i) line[(long long)(left + 1 + i) * stride] = e;
        return;
    }
    const int total = left + len + right;
    int lp = left, rp = right;
    while (lp > 0 || rp > 0) {
        int old = total - rp - lp;
        old = ((old - 1) / (len - 1)) * (len - 1) + 1;
        old -= 1;
        if (lp > 0) {
            const int chunk = old < lp ? old : lp;
            const T edge = line[(long long)lp * stride];
            for (int j = 0; j < chunk; ++j)
                line[(long long)(lp - chunk + j) * stride] =
                    X<T>::sub(X<T>::mul(T(2), edge), line[(long long)(lp + chunk - j) * stride]);
            lp -= chunk;
        }
        if (rp > 0) {
            const int chunk = old < rp ? old : rp;
            const int start = total - rp - 2;
            const T edge = line[(long long)(total - rp - 1) * stride];
            const int dst = total - rp;
            for (int j = 0; j < chunk; ++j)
                line[(long long)(dst + j) * stride] =
                    X<T>::sub(X<T>::mul(T(2), edge), line[(long long)(start - j) * stride]);
            rp -= chunk;
        }
    }
}

// copy image b into the interior of its padded buffer (top/left margin 1)
template <typename T>
__global__ void k_pad_copy(const T* __restrict__ src, long long istride, T* dst, long long pstride, int m, int n,
                           int W, const ImgState* st) {
    pdl_sync();
    const int b = blockIdx.y;
    if (st && st[b].done) return;
    const long long N = (long long)m * n;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), k = (int)(e % n);
        dst[(long long)b * pstride + (long long)(i + 1) * W + (k + 1)] = src[(long long)b * istride + e];
    }
}

// axis 0 (rows) over the original columns, then axis 1 over every padded row
template <typename T>
__global__ void k_pad_axis(T* buf, long long pstride, int axis, int m, int n, int H, int W, int bot, int rgt,
                           const ImgState* st) {
    pdl_sync();
    const int b = blockIdx.y;
    if (st && st[b].done) return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    T* base = buf + (long long)b * pstride;
    if (axis == 0) {
        if (t >= n) return;
        reflect_line(base + (t + 1), (long long)W, 1, m, bot);
    } else {
        if (t >= H) return;
        reflect_line(base + (long long)t * W, 1LL, 1, n, rgt);
    }
}

}  // namespace cmg
