// cmg_l1.cuh -- the level-1 visit (driver.sweep_layer with side 1,
// driver.py:225-251) as one fused four-colour tile kernel.
//
// Level 1 is the hot kernel: every pixel is a patch, eight tangent planes of
// its 3x3 neighbourhood (tangent.py:296-309) per pixel and colour.  A CTA owns
// a TH x TW pixel tile, stages the tile plus a 4-pixel halo (3 colours of
// dependency cone + the 1-pixel stencil ring) of u and f in shared
// memory, runs the four colour phases there and writes the tile to the output
// buffer (u_in -> u_out, so neighbouring CTAs keep reading pristine u_in).
//
// Shared memory is "quad-planar": pixel (2i+p, 2k+q) of the region lives in
// plane (p,q) at [i][k].  A colour phase updates exactly one plane, so a warp
// reads/writes consecutive words (no bank conflicts) and every neighbour of a
// pixel is at a compile-time offset in another plane.  Pixels outside the
// image that the stencil reaches (row -1 / m, column -1 / n) hold the odd
// reflection 2*edge - mirror (tangent.py:262-269), recomputed after every
// phase on border tiles.
#pragma once

#include "cmg_kernels.cuh"

namespace cmg {

template <typename T, int TH, int TW>
struct L1Geom {
    static constexpr int HALO = 4;
    static constexpr int RH = TH + 2 * HALO, RW = TW + 2 * HALO;  // region (even sizes)
    static constexpr int QH = RH / 2, QW = RW / 2;
    static constexpr int PLANE = QH * QW;
    static_assert(TH % 2 == 0 && TW % 2 == 0, "even tiles keep the colour parity");
    __device__ static constexpr int idx(int i, int k) {
        return ((i & 1) * 2 + (k & 1)) * PLANE + (i >> 1) * QW + (k >> 1);
    }
};

// Value of the 3x3 neighbourhood in the quad-planar region: dr,dc in {-1,0,1}
// relative to pixel (2qi+p, 2qk+q).
template <typename T, int TH, int TW, int P, int Q>
struct QuadAcc {
    using G = L1Geom<T, TH, TW>;
    const T* s;
    int qi, qk;
    template <int DR, int DC>
    __device__ __forceinline__ T at() const {
        constexpr int rp = (P + DR) & 1, cq = (Q + DC) & 1;
        constexpr int a = (P + DR) >> 1, b = (Q + DC) >> 1;  // arithmetic shift: -1 >> 1 == -1
        constexpr int off = (rp * 2 + cq) * G::PLANE + a * G::QW + b;
        return s[qi * G::QW + qk + off];
    }
};

// closed-form mean-curvature correction at level 1; pairs
// E-W / N-S (|p|^2=1) and the two diagonals (|p|^2=2)
template <typename T>
__device__ __forceinline__ T l1_chalf_fast(T c, T E, T W, T N, T S, T NE, T NW, T SE, T SW) {
    const T two = T(2);
    auto pair = [&](T up, T um, T uq, T umq, T fourL) {
        const T sp = up + um;
        const T Nn = sp - two * c;
        const T D = up - um;
        const T base = D * D + fourL;
        const T Sa = sp - two * uq, Sb = sp - two * umq;
        return Nn * (frsqrt(Sa * Sa + base) + frsqrt(Sb * Sb + base));
    };
    const T t1 = pair(E, W, N, S, T(4));
    const T t2 = pair(N, S, W, E, T(4));
    const T t3 = pair(NE, SW, NW, SE, T(8));
    const T t4 = pair(NW, SE, SW, NE, T(8));
    constexpr double SQRT2 = 1.4142135623730950488;
    return ((t1 + t2) + T(SQRT2) * (t3 + t4)) * T(0.125);
}

// backward-step constants of level 1 hoisted out of the pixel loop
template <typename T>
struct L1Back {
    int inner;
    T w, den, inv;
    const SolveParams* P;
};

template <typename T, int TH, int TW, int P, int Q, int MODE, int PREC>
__device__ __forceinline__ T l1_correction(const QuadAcc<T, TH, TW, P, Q>& A, T fval, const L1Back<T>& bk,
                                           int single) {
    using O = X<T>;
    const T c = A.template at<0, 0>();
    const T E = A.template at<0, 1>(), W = A.template at<0, -1>();
    const T N = A.template at<-1, 0>(), S = A.template at<1, 0>();
    const T NE = A.template at<-1, 1>(), NW = A.template at<-1, -1>();
    const T SE = A.template at<1, 1>(), SW = A.template at<1, -1>();
    // f* of a 1x1 patch: f - u (driver.py:244-246)
    const T fstar = O::sub(fval, c);
    T chalf;
    if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        chalf = l1_chalf_fast<T>(c, E, W, N, S, NE, NW, SE, SW);
    } else {
        // exact plane loop over compile-time offsets (tangent.py:296-309)
        auto U = [&](int dr, int dc) -> T {
            // dr, dc are compile-time after unrolling; map to the named values
            if (dr == 0 && dc == 0) return c;
            if (dr == 0 && dc == 1) return E;
            if (dr == 0 && dc == -1) return W;
            if (dr == -1 && dc == 0) return N;
            if (dr == 1 && dc == 0) return S;
            if (dr == -1 && dc == 1) return NE;
            if (dr == -1 && dc == -1) return NW;
            if (dr == 1 && dc == 1) return SE;
            return SW;
        };
        struct Acc9 {
            const decltype(U)& f;
            __device__ __forceinline__ T operator()(int i, int k) const { return f(i, k); }
        } acc{U};
        if constexpr (MODE == MODE_MEAN) {
            T d[8];
            static_for<0, 8>([&](auto l) { plane_exact<T, decltype(l)::value>(acc, 0, 0, c, &d[decltype(l)::value], nullptr); });
            T sum;
            if (single) {
                T tmp[8];
#pragma unroll
                for (int l = 0; l < 8; ++l) tmp[l] = d[l];
                sum = pairwise_of<T>(tmp, 8);
            } else {
                sum = d[0];
#pragma unroll
                for (int l = 1; l < 8; ++l) sum = O::add(sum, d[l]);
            }
            chalf = div_pow2<T, 8>(sum);
        } else {
            T v[8];
            static_for<0, 8>([&](auto l) { plane_exact<T, decltype(l)::value>(acc, 0, 0, c, nullptr, &v[decltype(l)::value]); });
            int imin = 0, imax = 0;
            bool nanseen = isnan(v[0]);
#pragma unroll
            for (int l = 1; l < 8; ++l) {
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
            for (int l = 1; l < 8; ++l) {
                if (l == imin) vmin = v[l];
                if (l == imax) vmax = v[l];
            }
            const int star = (fabs(vmin) <= fabs(vmax)) ? imin : imax;
            T ph = T(0);
            static_for<0, 8>([&](auto l) {
                if (star == decltype(l)::value) plane_exact<T, decltype(l)::value>(acc, 0, 0, c, &ph, nullptr);
            });
            chalf = ph;
        }
    }
    // backward steps (fbs.py:84-90); c_0 = 0 so the first step is (c_half + w f*)/(2+w)
    if (bk.inner == 1) {
        if constexpr (PREC == PREC_FAST)
            return (chalf + bk.w * fstar) * bk.inv;
        else
            return O::div(O::add(chalf, O::mul(bk.w, fstar)), bk.den);
    }
    T cc = T(0);
    for (int t = 0; t < bk.inner; ++t)
        cc = O::div(O::add(O::add(cc, chalf), O::mul(T(bk.P->w[1][t]), fstar)), T(bk.P->den[1][t]));
    return cc;
}

// refresh the reflected cells (row -1 / m, column -1 / n) of a border tile
template <typename T, int TH, int TW>
__device__ __forceinline__ void l1_reflect_fix(T* su, int r0, int c0, int m, int n) {
    using G = L1Geom<T, TH, TW>;
    // rows first (for in-image columns), then columns for every needed row
    const int rows[2] = {-1, m};
    for (int t = threadIdx.x; t < 2 * G::RW; t += blockDim.x) {
        const int ri = rows[t / G::RW];
        const int k = t % G::RW;
        const int i = ri - r0, gk = c0 + k;
        if (i < 0 || i >= G::RH || gk < 0 || gk >= n) continue;
        const int e = ri < 0 ? 0 : m - 1;
        const int mi = ri < 0 ? 1 : m - 2;
        su[G::idx(i, k)] = X<T>::sub(X<T>::mul(T(2), su[G::idx(e - r0, k)]), su[G::idx(mi - r0, k)]);
    }
    __syncthreads();
    const int cols[2] = {-1, n};
    for (int t = threadIdx.x; t < 2 * G::RH; t += blockDim.x) {
        const int ck = cols[t / G::RH];
        const int i = t % G::RH;
        const int k = ck - c0, gi = r0 + i;
        if (k < 0 || k >= G::RW || gi < -1 || gi > m) continue;
        const int e = ck < 0 ? 0 : n - 1;
        const int mk = ck < 0 ? 1 : n - 2;
        su[G::idx(i, k)] = X<T>::sub(X<T>::mul(T(2), su[G::idx(i, e - c0)]), su[G::idx(i, mk - c0)]);
    }
    __syncthreads();
}

// Energy terms of the tile's owned pixels from the staged (pristine) region:
// level-1 curvature from the 3x3 neighbourhood (closed form, as k_energy),
// fidelity from sf, |u - u_prev| and (u - ref)^2 from global memory; fp64
// accumulation; CTA sums -> partials (tangent.energy, tangent.py:325-341;
// driver.py:284-291, :161-166)
template <typename T, int TH, int TW>
__device__ __forceinline__ void l1_energy_sums(const T* su, const T* sf, int R, int C, int m, int n, const T* up,
                                               const T* rf, int mode, double* partials, int b, int cta, int nbx) {
    using G = L1Geom<T, TH, TW>;
    // owned pixels plane by plane (colour class (P,Q) of the quad-planar layout):
    // every neighbour is a compile-time offset from one shared-memory base
    constexpr int PH = TH / 2, PW = TW / 2, CNT = PH * PW;
    static_assert(G::HALO % 2 == 0, "owned pixels start on an even region row");
    double acc[NSUM] = {0, 0, 0, 0, 0};
    // fully unrolled (2 pixels per plane and thread for 32 x 64 tiles): the u_prev
    // loads of all of a thread's pixels are issued before the first use
    static_for<0, 4>([&](auto cp) {
        constexpr int P = decltype(cp)::value >> 1, Q = decltype(cp)::value & 1;
#pragma unroll
        for (int it = 0; it < (CNT + 255) / 256; ++it) {
            const int t = threadIdx.x + it * 256;
            if (CNT % 256 != 0 && t >= CNT) continue;
            const int ii = t / PW, kk = t % PW;
            const int gi = R + 2 * ii + P, gk = C + 2 * kk + Q;
            if (gi >= m || gk >= n) continue;
            const QuadAcc<T, TH, TW, P, Q> A{su, G::HALO / 2 + ii, G::HALO / 2 + kk};
            const T c = A.template at<0, 0>();
            const T tm = curv_term<T>(c, A.template at<0, 1>(), A.template at<0, -1>(), A.template at<-1, 0>(),
                                      A.template at<1, 0>(), A.template at<-1, 1>(), A.template at<1, -1>(),
                                      A.template at<-1, -1>(), A.template at<1, 1>(), mode);
            const long long g = (long long)gi * n + gk;
            const double c64 = (double)c;
            const double d = c64 - (double)sf[(P * 2 + Q) * G::PLANE + (G::HALO / 2 + ii) * G::QW + G::HALO / 2 + kk];
            acc[0] += (double)tm;
            acc[1] += d * d;
            acc[2] += fabs(c64 - (double)up[g]);
            acc[3] += fabs(c64);
            if (rf) {
                const double dr = c64 - (double)rf[g];
                acc[4] += dr * dr;
            }
        }
    });
    cta_sums_store(acc, partials, nbx, cta, b);
}

// branch-free exact correction (cmg_l1loop.cuh)
template <int TH, int TW, int C>
__device__ __forceinline__ double l1_correction_unrolled(const double* sp, double fval, double w, double den,
                                                         unsigned guard);

// (mean mode: 4 CTAs of 256 threads per SM, <= 64 registers)
// LOOP: fp64 exact mean mode with one inner iteration and no single-patch colour
// class -- the branch-free pixel code of cmg_l1loop.cuh
template <typename T, int MODE, int PREC, int TH, int TW, bool LOOP = false>
__global__ void __launch_bounds__(256, MODE == MODE_MEAN ? 4 : 1) k_l1_tile(FusedArgs<T> a) {
    pdl_sync();
    using G = L1Geom<T, TH, TW>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* su = reinterpret_cast<T*>(smem_raw);
    T* sf = su + 4 * G::PLANE;
    const int b = blockIdx.z;
    const int tr = blockIdx.y, tc = blockIdx.x;
    const int R = tr * TH, C = tc * TW;
    const T* uin = a.uin + (long long)b * a.istride;
    const T* f = a.f + (long long)b * a.istride;
    T* uout = a.uout + (long long)b * a.istride;
    const int m = a.m, n = a.n;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x, nbx = gridDim.x * gridDim.y;
    if (a.st[b].done) {  // stopped image (its final u stays in ImgState::final_buf)
        if (a.efuse) efused_ticket(a.fz, a.partials, nbx, b, reinterpret_cast<double*>(smem_raw));
        return;
    }
    const int r0 = R - G::HALO, c0 = C - G::HALO;
    const bool border = (r0 < 1) || (c0 < 1) || (r0 + G::RH >= m) || (c0 + G::RW >= n);
    // stage u and f
    if (!border && (n & 1) == 0) {
        // interior tile: every load of the thread (column pairs, 2 x sizeof(T) bytes) is
        // issued before the first shared-memory store -- one memory round trip instead
        // of one per element (the bounds-checked loop below serialises them)
        struct alignas(2 * sizeof(T)) Pair {
            T a, b;
        };
        constexpr int PW = G::RW / 2, PAIRS = G::RH * PW, IT = (PAIRS + 255) / 256;
        Pair vu[IT], vf[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 256;
            if (PAIRS % 256 == 0 || it + 1 < IT || e < PAIRS) {
                const int i = e / PW, kp = e % PW;
                const long long g = (long long)(r0 + i) * n + c0 + 2 * kp;
                vu[it] = *reinterpret_cast<const Pair*>(uin + g);
                vf[it] = *reinterpret_cast<const Pair*>(f + g);
            }
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 256;
            if (PAIRS % 256 == 0 || it + 1 < IT || e < PAIRS) {
                const int i = e / PW, kp = e % PW;
                const int base = ((i & 1) * 2) * G::PLANE + (i >> 1) * G::QW + kp;  // idx(i, 2 kp)
                su[base] = vu[it].a;
                su[base + G::PLANE] = vu[it].b;
                sf[base] = vf[it].a;
                sf[base + G::PLANE] = vf[it].b;
            }
        }
    } else {
        // border tile: in-image cells of the region
        for (int e = threadIdx.x; e < G::RH * G::RW; e += blockDim.x) {
            const int i = e / G::RW, k = e % G::RW;
            const int gi = r0 + i, gk = c0 + k;
            if (gi >= 0 && gi < m && gk >= 0 && gk < n) {
                const long long g = (long long)gi * n + gk;
                su[G::idx(i, k)] = uin[g];
                sf[G::idx(i, k)] = f[g];
            }
        }
    }
    __syncthreads();
    if (border) l1_reflect_fix<T, TH, TW>(su, r0, c0, m, n);
    if (a.efuse)
        l1_energy_sums<T, TH, TW>(su, sf, R, C, m, n, a.uprev + (long long)b * a.istride,
                                  a.ref ? a.ref + (long long)b * a.istride : nullptr, a.mode, a.partials, b, cta,
                                  nbx);
    bool bad = false;
    // four always-set bits from unrelated runtime values (cmg_l1loop.cuh: plane-pair guards)
    const unsigned guard = (m > 0 ? 1u : 0u) | (n > 0 ? 2u : 0u) | (a.istride >= 0 ? 4u : 0u) | (nbx > 0 ? 8u : 0u);
    L1Back<T> bk;
    bk.P = a.P;
    bk.inner = a.P->inner;
    bk.w = T(a.P->w[1][0]);
    bk.den = T(a.P->den[1][0]);
    bk.inv = T(1.0 / a.P->den[1][0]);
    static_for<0, 4>([&](auto cphase) {
        constexpr int c = decltype(cphase)::value;
        constexpr int P = c >> 1, Q = c & 1;
        constexpr int h = 3 - c;
        // region-relative pixel rows i in [HALO-h, HALO+TH+h) with i = P (mod 2)
        constexpr int i_lo = G::HALO - h + (((G::HALO - h) & 1) != P ? 1 : 0);
        constexpr int i_hi = G::HALO + TH + h;
        constexpr int k_lo = G::HALO - h + (((G::HALO - h) & 1) != Q ? 1 : 0);
        constexpr int k_hi = G::HALO + TW + h;
        constexpr int NI = (i_hi - i_lo + 1) / 2, NK = (k_hi - k_lo + 1) / 2;
        constexpr int CNT = NI * NK;
        constexpr int ITERS = (CNT + 255) / 256;
        const int single = (a.hc[c] * a.wc[c] == 1);
        // one copy of the pixel code per colour phase (not per iteration): the
        // fully unrolled exact kernel overflowed the instruction cache
#pragma unroll 1
        for (int it = 0; it < ITERS; ++it) {
            const int t = threadIdx.x + it * 256;
            if (CNT % 256 == 0 || it + 1 < ITERS || t < CNT) {
                const int ii = t / NK, kk = t % NK;
                const int qi = (i_lo >> 1) + ii, qk = (k_lo >> 1) + kk;
                bool ok = true;
                if (border) {
                    const int gi = r0 + 2 * qi + P, gk = c0 + 2 * qk + Q;
                    ok = gi >= 0 && gi < m && gk >= 0 && gk < n;
                }
                if (ok) {
                    QuadAcc<T, TH, TW, P, Q> A{su, qi, qk};
                    const int sidx = (P * 2 + Q) * G::PLANE + qi * G::QW + qk;
                    T corr;
                    if constexpr (LOOP)
                        corr = l1_correction_unrolled<TH, TW, c>(su + qi * G::QW + qk, sf[sidx], bk.w, bk.den, guard);
                    else
                        corr = l1_correction<T, TH, TW, P, Q, MODE, PREC>(A, sf[sidx], bk, single);
                    bad |= !isfinite(corr);
                    su[sidx] = X<T>::add(su[sidx], corr);
                }
            }
        }
        __syncthreads();
        if (border) l1_reflect_fix<T, TH, TW>(su, r0, c0, m, n);
    });
    if (__syncthreads_or(bad) && threadIdx.x == 0) {
        if (a.efuse) {
            a.st[b].bad1 = 1;
            __threadfence();  // visible to the CTA that finalizes (efused_ticket)
        } else {
            a.st[b].bad = 1;
        }
    }
    for (int e = threadIdx.x; e < TH * TW; e += blockDim.x) {
        const int i = e / TW, k = e % TW;
        const int gi = R + i, gk = C + k;
        if (gi < m && gk < n) uout[(long long)gi * n + gk] = su[G::idx(i + G::HALO, k + G::HALO)];
    }
    if (a.efuse) {
        __syncthreads();  // shared memory becomes the finalize scratch
        efused_ticket(a.fz, a.partials, nbx, b, reinterpret_cast<double*>(smem_raw));
    }
}

}  // namespace cmg
