// cmg_coarse.cuh -- fused four-colour visit of levels 2 and 3 (patch sides 3
// and 7; driver.sweep_layer, driver.py:225-251) in shared memory.
//
// A CTA owns TP x TP patches.  It stages their pixels plus a halo of 3
// patches and a 1-pixel ring (the stencil reaches one pixel past a
// patch, so the dependency cone grows one patch per colour), runs the four
// colour phases with compile-time patch counts, and writes its own patches to
// the output buffer (u_in -> u_out).  TS lanes cooperate on a patch:
//   TS == 1: one thread per patch, every plane offset a compile-time constant;
//   TS  > 1: lane t owns patch row t for f* and the update, planes are split
//            over lanes through a shared-memory table of linearised offsets,
//            and the NumPy-ordered reductions are replayed with shuffles.
// Arithmetic is exactly that of the per-colour kernels (exact or fast).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors are built on the host)

#include "cmg_kernels.cuh"

namespace cmg {

template <typename T, int LAYER, int TP>
struct CoarseGeom {
    static constexpr int S = (1 << LAYER) - 1;
    static constexpr int R = 1 << (LAYER - 1);
    static constexpr int NPL = 1 << (LAYER + 2);
    static constexpr int HALO_P = 3;
    static constexpr int RD = (TP + 2 * HALO_P) * S + 2;  // region side (pixels)
    // TMA boxes must start on a 16-byte column boundary: the box is widened by
    // up to VEC-1 columns and the region starts `sh` columns into each row
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int BW = (RD + VEC - 1 + VEC - 1) / VEC * VEC;  // box width (columns)
    static constexpr int LD = BW;                                    // dense rows: the TMA box layout
    static constexpr int CELLS = RD * LD;
    static constexpr int CELLS_AL = (CELLS * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);  // 128-B aligned
};

// ---- TMA (cp.async.bulk.tensor) staging -----------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 3-D box {x = column, y = row, z = image} -> shared memory (dense x-fastest)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// shared-memory accessor with compile-time-friendly addressing: pixel
// (R0 + dr, C0 + dc) of the image -> su[base + dr*LD + dc]
template <typename T, int LD>
struct SBase {
    const T* s;
    int base;  // offset of the patch's top-left pixel
    __device__ __forceinline__ T operator()(int dr, int dc) const { return s[base + dr * LD + dc]; }
};

// odd-reflection view for border tiles (image coordinates relative to the
// region origin); reflections read in-image cells of the region only
template <typename T, int LD>
struct SRefl {
    const T* s;
    int r0, c0, m, n;
    __device__ __forceinline__ T at(int i, int k) const { return s[(i - r0) * LD + (k - c0)]; }
    __device__ __forceinline__ T row(int i, int k) const {
        if (i >= 0 && i < m) return at(i, k);
        const int e = (i < 0) ? 0 : m - 1;
        const int mi = (i < 0) ? -i : 2 * (m - 1) - i;
        return X<T>::sub(X<T>::mul(T(2), at(e, k)), at(mi, k));
    }
    __device__ __forceinline__ T operator()(int i, int k) const {
        if (k >= 0 && k < n) return row(i, k);
        const int e = (k < 0) ? 0 : n - 1;
        const int mk = (k < 0) ? -k : 2 * (n - 1) - k;
        return X<T>::sub(X<T>::mul(T(2), row(i, e)), row(i, mk));
    }
};

// Border tiles: materialise the padded values the stencil/f* can read
// (rows -1..mp and columns -1..np of the level) inside the region, so the
// phase code can read the region as if the image were larger.
template <typename T, int LAYER, int TP>
__device__ __forceinline__ void coarse_fill_pad(T* s, int r0, int c0, int m, int n, int mp, int np) {
    using G = CoarseGeom<T, LAYER, TP>;
    // cells outside the image but inside [-1, mp] x [-1, np]: odd reflection
    SRefl<T, G::LD> A{s, r0, c0, m, n};
    // rows first: pad rows over in-image columns
    for (int e = threadIdx.x; e < G::RD * G::RD; e += blockDim.x) {
        const int i = e / G::RD, k = e % G::RD;
        const int gi = r0 + i, gk = c0 + k;
        if (gi >= -1 && gi <= mp && (gi < 0 || gi >= m) && gk >= 0 && gk < n) s[i * G::LD + k] = A.row(gi, gk);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < G::RD * G::RD; e += blockDim.x) {
        const int i = e / G::RD, k = e % G::RD;
        const int gi = r0 + i, gk = c0 + k;
        if (gi >= -1 && gi <= mp && gk >= -1 && gk <= np && (gk < 0 || gk >= n)) {
            const int ee = (gk < 0) ? 0 : n - 1;
            const int mk = (gk < 0) ? -gk : 2 * (n - 1) - gk;
            s[i * G::LD + k] = X<T>::sub(X<T>::mul(T(2), s[i * G::LD + (ee - c0)]), s[i * G::LD + (mk - c0)]);
        }
    }
    __syncthreads();
}

// ---- plane offset table (linearised: dr*LD + dc) for TS > 1 -------------
struct PlaneLin {
    int ox, oy, oz;            // linear offsets of the three vertices
    signed char x0, x1, y0, y1, z0, z1, pad0, pad1;
};

// ---- one patch, TS == 1 (compile-time offsets) ---------------------------
template <typename T, int LAYER, int MODE, int PREC, class Acc>
__device__ __forceinline__ T coarse_solve_thread(const Acc& U, const Acc& F, const SweepArgs<T>& a, T w, T den,
                                                 T inv, const double* fsp = nullptr) {
    using O = X<T>;
    constexpr int S = (1 << LAYER) - 1, R = 1 << (LAYER - 1), NPL = 1 << (LAYER + 2);
    T acc;
    if (MODE == MODE_MEAN && PREC == PREC_FAST && fsp) {  // f* from the precomputed sum of f (fast mode)
        T us = T(0);
#pragma unroll
        for (int aa = 0; aa < S; ++aa)
#pragma unroll
            for (int bb = 0; bb < S; ++bb) us += U(aa, bb);
        acc = T(__ldg(fsp) - (double)us);
    } else if (a.flat) {
        acc = fstar_flat_sum<T, S>(U, F, 0, 0);
    } else {
        acc = T(0);
#pragma unroll
        for (int aa = 0; aa < S; ++aa)
            acc = O::add(acc, pairwise_small<T>(S, [&](int bb) { return O::sub(F(aa, bb), U(aa, bb)); }));
    }
    const T fstar = O::div(acc, T(S * S));
    const int ci = R - 1, cc = R - 1;
    const T uo = U(ci, cc);
    T chalf;
    if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        T sum = T(0);
        static_for<0, NPL / 2>([&](auto k) { sum += pair_fast<T, decltype(k)::value>(U, ci, cc, uo); });
        chalf = sum * T(1.0 / NPL);
    } else if constexpr (MODE == MODE_MEAN) {
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
    } else {
        T v[NPL];
        static_for<0, NPL>([&](auto l) { plane_exact<T, decltype(l)::value>(U, ci, cc, uo, nullptr, &v[decltype(l)::value]); });
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
        T ph = T(0);
        static_for<0, NPL>([&](auto l) {
            if (star == decltype(l)::value) plane_exact<T, decltype(l)::value>(U, ci, cc, uo, &ph, nullptr);
        });
        chalf = ph;
    }
    if (a.P->inner == 1) {
        if constexpr (PREC == PREC_FAST)
            return (chalf + w * fstar) * inv;
        else
            return O::div(O::add(chalf, O::mul(w, fstar)), den);
    }
    T c = T(0);
    for (int t = 0; t < a.P->inner; ++t)
        c = O::div(O::add(O::add(c, chalf), O::mul(T(a.P->w[LAYER][t]), fstar)), T(a.P->den[LAYER][t]));
    return c;
}

// ---- one patch, TS > 1 lanes (shared-memory plane table) -----------------
template <typename T, int LAYER, int MODE, int PREC, int TS>
__device__ __forceinline__ T coarse_solve_team(const T* su, const T* sf, int base, int lane, const PlaneLin* tab,
                                               int ld, const SweepArgs<T>& a, T w, T den, T inv) {
    using O = X<T>;
    constexpr int S = (1 << LAYER) - 1, R = 1 << (LAYER - 1), NPL = 1 << (LAYER + 2);
    constexpr unsigned FULL = 0xffffffffu;
    static_assert(TS >= S && (32 % TS) == 0, "team size");
    // f*: lane t < S sums row t pairwise; rows accumulate sequentially
    T rowsum = T(0);
    if (a.flat) {
        if (lane == 0) {
            rowsum = O::add(T(0), pairwise_small<T>(S * S, [&](int e) {
                const int o = base + (e / S) * ld + (e % S);
                return O::sub(sf[o], su[o]);
            }));
        }
    } else if (lane < S) {
        const int ro = base + lane * ld;
        rowsum = pairwise_small<T>(S, [&](int bb) { return O::sub(sf[ro + bb], su[ro + bb]); });
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
    const int cidx = base + (R - 1) * ld + (R - 1);
    const T uo = su[cidx];
    T chalf;
    if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        constexpr int NPAIR = NPL / 2;
        T part = T(0);
#pragma unroll
        for (int k = 0; k < (NPAIR + TS - 1) / TS; ++k) {
            const int pi = lane + k * TS;
            if (pi < NPAIR) {
                const PlaneLin pl = tab[2 * pi];
                const int Lq = pl.x0 * pl.x0 + pl.x1 * pl.x1;
                const T up = su[cidx + pl.ox], um = su[cidx - pl.ox];
                const T uq = su[cidx + pl.oy], umq = su[cidx - pl.oy];
                const T sp = up + um;
                const T N = sp - T(2) * uo;
                const T Dd = up - um;
                const T bse = Dd * Dd + T(4 * Lq);
                const T Sa = sp - T(2) * uq, Sb = sp - T(2) * umq;
                part += (sqrt(T(Lq)) * N) * (frsqrt(Sa * Sa + bse) + frsqrt(Sb * Sb + bse));
            }
        }
#pragma unroll
        for (int o = TS / 2; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o, TS);
        chalf = part * T(1.0 / NPL);
    } else {
        struct Lin {
            const T* s;
            int c;
            int ld;
            __device__ __forceinline__ T operator()(int i, int k) const { return s[c + i * ld + k]; }
        } L{su, cidx, ld};
        constexpr int PPL = NPL / TS;
        if constexpr (MODE == MODE_MEAN) {
            T d[PPL];
#pragma unroll
            for (int k = 0; k < PPL; ++k) {
                const PlaneLin pl = tab[lane + k * TS];
                plane_exact_rt<T>(L, 0, 0, uo, PlaneRT{pl.x0, pl.x1, pl.y0, pl.y1, pl.z0, pl.z1}, &d[k], nullptr);
            }
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
            ArgBest<T> bmin, bmax;
#pragma unroll
            for (int k = 0; k < PPL; ++k) {
                const PlaneLin pl = tab[lane + k * TS];
                T v;
                plane_exact_rt<T>(L, 0, 0, uo, PlaneRT{pl.x0, pl.x1, pl.y0, pl.y1, pl.z0, pl.z1}, nullptr, &v);
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
            if (lane == 0) {
                const PlaneLin pl = tab[star];
                plane_exact_rt<T>(L, 0, 0, uo, PlaneRT{pl.x0, pl.x1, pl.y0, pl.y1, pl.z0, pl.z1}, &ph, nullptr);
            }
            chalf = __shfl_sync(FULL, ph, 0, TS);
        }
    }
    if (a.P->inner == 1) {
        if constexpr (PREC == PREC_FAST)
            return (chalf + w * fstar) * inv;
        else
            return O::div(O::add(chalf, O::mul(w, fstar)), den);
    }
    T c = T(0);
    for (int t = 0; t < a.P->inner; ++t)
        c = O::div(O::add(O::add(c, chalf), O::mul(T(a.P->w[LAYER][t]), fstar)), T(a.P->den[LAYER][t]));
    return c;
}

// FS: fast mean mode with per-patch f sums (a.fsum): f is not staged at all
template <typename T, int LAYER, int MODE, int PREC, int TP, int TS, int NT, bool FS = false>
__global__ void __launch_bounds__(NT) k_coarse_tile(FusedArgs<T> a, const __grid_constant__ CUtensorMap tmu,
                                                    const __grid_constant__ CUtensorMap tmf, int use_tma) {
    static_assert(!FS || (TS == 1 && MODE == MODE_MEAN && PREC == PREC_FAST), "f sums: one thread per patch, fast");
    pdl_sync();
    using G = CoarseGeom<T, LAYER, TP>;
    constexpr int S = G::S, RD = G::RD, LD = G::LD;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TMA destinations must be 128-byte aligned: align the carve-up explicitly
    unsigned char* base128 = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
    T* su_al = reinterpret_cast<T*>(base128);
    T* sf_al = su_al + G::CELLS_AL;
    PlaneLin* tab = reinterpret_cast<PlaneLin*>(su_al + (FS ? 1 : 2) * G::CELLS_AL);
    unsigned long long* mbarp = reinterpret_cast<unsigned long long*>(tab + G::NPL + (G::NPL & 1));
    const int b = blockIdx.z;
    const int P0 = blockIdx.y * TP, Q0 = blockIdx.x * TP;
    const int r0 = (P0 - G::HALO_P) * S - 1, c0 = (Q0 - G::HALO_P) * S - 1;
    const int sh = ((c0 % G::VEC) + G::VEC) % G::VEC;  // region column 0 sits sh columns into a box row
    T* su = su_al + sh;
    T* sf = sf_al + sh;
    const T* uin = a.uin + (long long)b * a.istride;
    const T* f = a.f + (long long)b * a.istride;
    T* uout = a.uout + (long long)b * a.istride;
    const int m = a.m, n = a.n;
    const int ti0 = P0 * S, ti1 = min((P0 + TP) * S, m);
    const int tk0 = Q0 * S, tk1 = min((Q0 + TP) * S, n);
    if (a.st[b].done) return;  // stopped image (final u in ImgState::final_buf)
    if constexpr (TS > 1) {
        for (int l = threadIdx.x; l < G::NPL; l += NT) {
            const PlaneRT q = PlaneRT::getg(l);
            PlaneLin p;
            p.x0 = q.x0;
            p.x1 = q.x1;
            p.y0 = q.y0;
            p.y1 = q.y1;
            p.z0 = q.z0;
            p.z1 = q.z1;
            p.ox = p.x0 * LD + p.x1;
            p.oy = p.y0 * LD + p.y1;
            p.oz = p.z0 * LD + p.z1;
            tab[l] = p;
        }
    }
    // TMA only for boxes fully inside the image (negative box coordinates
    // trap on this driver); border tiles stage with plain loads
    const bool inside_box = (r0 >= 0) && (c0 - sh >= 0) && (r0 + RD <= m) && (c0 - sh + G::BW <= n);
    if (use_tma && inside_box) {
        // one elected thread moves the whole region (u and f) with TMA
        if (threadIdx.x == 0) mbar_init(mbarp, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_expect_tx(mbarp, (FS ? 1u : 2u) * RD * G::BW * (unsigned)sizeof(T));
            tma_load_3d(su_al, &tmu, c0 - sh, r0, b, mbarp);
            if (!FS) tma_load_3d(sf_al, &tmf, c0 - sh, r0, b, mbarp);
        }
        mbar_wait(mbarp, 0);
    } else {
        // stage the in-image part of the region (rows by warps, coalesced)
        for (int i = threadIdx.x / 32; i < RD; i += NT / 32) {
            const int gi = r0 + i;
            if (gi < 0 || gi >= m) continue;
            const T* ur = uin + (long long)gi * n;
            const T* fr = f + (long long)gi * n;
            for (int k = threadIdx.x & 31; k < RD; k += 32) {
                const int gk = c0 + k;
                if (gk >= 0 && gk < n) {
                    su[i * LD + k] = ur[gk];
                    if (!FS) sf[i * LD + k] = fr[gk];
                }
            }
        }
        __syncthreads();
    }
    const bool border = (r0 < 0) || (c0 < 0) || (r0 + RD > m) || (c0 + RD > n);
    const int mp = a.mj * S, np = a.nj * S;
    SweepArgs<T> sa;
    sa.m = m;
    sa.n = n;
    sa.layer = LAYER;
    sa.s = S;
    sa.r = 1 << (LAYER - 1);
    sa.P = a.P;
    sa.st = a.st;
    sa.dbg = 0;
    sa.bk.inner = a.P->inner;
    sa.bk.w0 = a.P->w[LAYER][0];
    sa.bk.den0 = a.P->den[LAYER][0];
    sa.bk.inv0 = 1.0 / sa.bk.den0;
    const T w = T(a.P->w[LAYER][0]), den = T(a.P->den[LAYER][0]), inv = T(1.0 / a.P->den[LAYER][0]);
    bool bad = false;
    // pad values of u are refreshed after every phase on border tiles; f's once
    if (border) {
        if (!FS) coarse_fill_pad<T, LAYER, TP>(sf, r0, c0, m, n, mp, np);
        coarse_fill_pad<T, LAYER, TP>(su, r0, c0, m, n, mp, np);
    }
    static_for<0, 4>([&](auto cphase) {
        constexpr int c = decltype(cphase)::value;
        constexpr int P = c >> 1, Q = c & 1;
        constexpr int h = 3 - c;
        // patch rows pa = P0 - h + 2*ia (+ parity fix), cols similarly; counts at most (TP + 2h + 1) / 2
        constexpr int NA = (TP + 2 * h + 1) / 2;
        constexpr int CNT = NA * NA;
        constexpr int NTEAMS = NT / TS;
        constexpr int ITERS = (CNT + NTEAMS - 1) / NTEAMS;
        const int alo = P0 - h + (((P0 - h) & 1) != P ? 1 : 0);
        const int blo = Q0 - h + (((Q0 - h) & 1) != Q ? 1 : 0);
        const int ahi = min(P0 + TP + h, a.mj), bhi = min(Q0 + TP + h, a.nj);
        sa.p = P;
        sa.q = Q;
        sa.hc = a.hc[c];
        sa.wc = a.wc[c];
        sa.flat = (sa.wc == 1);
        sa.single = (sa.hc * sa.wc == 1);
        const int team = threadIdx.x / TS, lane = threadIdx.x % TS;
#pragma unroll
        for (int it = 0; it < ITERS; ++it) {
            int t = team + it * NTEAMS;
            // warp-uniform skip of fully idle warps; teams inside a warp stay converged
            const int warp_first = ((threadIdx.x & ~31) / TS) + it * NTEAMS;
            if (warp_first >= CNT) break;
            const int pa = alo + 2 * (t / NA), pb = blo + 2 * (t % NA);
            bool valid = t < CNT && pa >= 0 && pa < ahi && pb >= 0 && pb < bhi;
            const int R0 = valid ? pa * S : P0 * S, C0 = valid ? pb * S : Q0 * S;  // safe base when idle
            const int base = (R0 - r0) * LD + (C0 - c0);
            T cv;
            if constexpr (TS == 1) {
                SBase<T, LD> U{su, base}, F{sf, base};
                const double* fsp = FS ? a.fsum + b * a.fs_img + (long long)pa * a.fs_ld + pb : nullptr;
                if (valid) cv = coarse_solve_thread<T, LAYER, MODE, PREC>(U, F, sa, w, den, inv, fsp);
            } else {
                cv = coarse_solve_team<T, LAYER, MODE, PREC, TS>(su, sf, base, lane, tab, LD, sa, w, den, inv);
            }
            if (valid) {
                if (lane == 0) bad |= !isfinite(cv);
                // apply to the in-image pixels of the patch (lane t: rows t, t+TS, ...)
                for (int rr = lane; rr < S; rr += TS) {
                    if (R0 + rr >= m) break;
#pragma unroll
                    for (int cc2 = 0; cc2 < S; ++cc2) {
                        if (C0 + cc2 < n) {
                            T* pp = su + base + rr * LD + cc2;
                            *pp = X<T>::add(*pp, cv);
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (border) coarse_fill_pad<T, LAYER, TP>(su, r0, c0, m, n, mp, np);
    });
    if (__syncthreads_or(bad) && threadIdx.x == 0) a.st[b].bad = 1;
    for (int i = ti0 + threadIdx.x / 32; i < ti1; i += NT / 32)
        for (int k = tk0 + (threadIdx.x & 31); k < tk1; k += 32)
            uout[(long long)i * n + k] = su[(i - r0) * LD + (k - c0)];
}

}  // namespace cmg
