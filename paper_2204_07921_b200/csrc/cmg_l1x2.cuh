// cmg_l1x2.cuh -- level-1 visit, fp32 fast mean-curvature path, with
// Blackwell packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2).
//
// Same tiling and semantics as k_l1_tile (four colour phases of a TH x TW tile
// + 4-pixel halo in quad-planar shared memory, u_in -> u_out), but every
// thread relaxes TWO same-colour pixels of one region row at once: in the
// quad-planar layout they are adjacent words of one plane, so their
// neighbourhoods load as 64-bit pairs and the closed-form distance sums
// run as f32x2 instructions -- half the FP issue slots per
// pixel.  The reciprocal square roots stay scalar MUFU.RSQ.
#pragma once

#include "cmg_l1.cuh"

namespace cmg {

struct F2 {
    unsigned long long v;
};

__device__ __forceinline__ F2 f2_pack(float lo, float hi) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(F2 a, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
}
__device__ __forceinline__ F2 f2_splat(float x) { return f2_pack(x, x); }
__device__ __forceinline__ F2 operator+(F2 a, F2 b) {
    F2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 operator-(F2 a, F2 b) {
    F2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
// Products are fma(a, b, nz) with nz = -0.0 held in a register loaded from a
// kernel argument: bitwise the rounded product, but ptxas can neither fold it
// to a multiply nor contract it with a neighbouring add.  (It does contract
// mul.rn.f32x2 + add.rn.f32x2, differently per call site, which made two code
// paths of the same formula differ by 1 ulp.)
__device__ __forceinline__ F2 mul2(F2 a, F2 b, F2 nz) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(nz.v));
    return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
// MUFU.RSQ without the subnormal-input fix-up of rsqrtf(): the arguments are
// S^2 + D^2 + 4|p|^2 >= 4 (never subnormal)
__device__ __forceinline__ float rsq_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ F2 rsqrt2(F2 a) {
    F2 r;  // one asm block so the halves stay in their register pair (no moves)
    asm("{\n\t.reg .f32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\trsqrt.approx.ftz.f32 lo, lo;\n\t"
        "rsqrt.approx.ftz.f32 hi, hi;\n\tmov.b64 %0, {lo, hi};\n\t}"
        : "=l"(r.v)
        : "l"(a.v));
    return r;
}
// reciprocal square root of a pair on the FMA pipe: bit-trick seed + 3 Newton
// steps in packed fp32 (relative error ~1e-7), used to balance the MUFU pipe
__device__ __forceinline__ F2 rsqrt2_nr(F2 a, F2 nz) {
    F2 y;
    asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tshr.u32 lo, lo, 1;\n\tshr.u32 hi, hi, 1;\n\t"
        "sub.u32 lo, 0x5f375a86, lo;\n\tsub.u32 hi, 0x5f375a86, hi;\n\tmov.b64 %0, {lo, hi};\n\t}"
        : "=l"(y.v)
        : "l"(a.v));
    const F2 mh = mul2(f2_splat(-0.5f), a, nz), c15 = f2_splat(1.5f);
#pragma unroll
    for (int it = 0; it < 3; ++it) y = mul2(y, fma2(mh, mul2(y, y, nz), c15), nz);
    return y;
}
__device__ __forceinline__ F2 lds2(const float* p) {
    F2 r;
    r.v = *reinterpret_cast<const unsigned long long*>(p);
    return r;
}

// closed-form level-1 c_half for two pixels (l1_chalf_fast, packed); NR > 0
// moves the diagonal pairs' rsqrt to the FMA pipe (balances MUFU)
template <int NR>
__device__ __forceinline__ F2 l1_chalf_x2(F2 c, F2 E, F2 W, F2 N, F2 S, F2 NE, F2 NW, F2 SE, F2 SW, F2 nz) {
    const F2 m2 = f2_splat(-2.f);
    const F2 four = f2_splat(4.f), eight = f2_splat(8.f);
    auto pair = [&](F2 up, F2 um, F2 uq, F2 umq, F2 fourL, auto nr) {
        const F2 sp = up + um;
        const F2 Nn = fma2(m2, c, sp);
        const F2 D = up - um;
        const F2 base = fma2(D, D, fourL);
        const F2 Sa = fma2(m2, uq, sp), Sb = fma2(m2, umq, sp);
        if constexpr (decltype(nr)::value)
            return mul2(Nn, rsqrt2_nr(fma2(Sa, Sa, base), nz) + rsqrt2_nr(fma2(Sb, Sb, base), nz), nz);
        else
            return mul2(Nn, rsqrt2(fma2(Sa, Sa, base)) + rsqrt2(fma2(Sb, Sb, base)), nz);
    };
    using NO = std::integral_constant<bool, false>;
    using YES = std::integral_constant<bool, (NR > 0)>;
    const F2 t1 = pair(E, W, N, S, four, NO{});
    const F2 t2 = pair(N, S, W, E, four, NO{});
    const F2 t3 = pair(NE, SW, NW, SE, eight, YES{});
    const F2 t4 = pair(NW, SE, SW, NE, eight, NO{});
    return mul2(fma2(f2_splat(1.41421356237309505f), t3 + t4, t1 + t2), f2_splat(0.125f), nz);
}

// Energy terms of the tile's owned pixels (energy-fused cycle, fp32 images):
// as l1_energy_sums, with f from shared memory or (FG) global memory; each
// thread adds its <= 7 pixels of a colour plane in fp32 (<= 6 ulp relative,
// the size of the fp32 per-pixel terms) before the fp64 accumulators
template <int TH, int TW, bool FG, int NTH>
__device__ __forceinline__ void x2_energy_sums(const float* su, const float* sf, const float* f, int R, int C,
                                               int m, int n, const float* up, const float* rf, double* partials,
                                               int b, int cta, int nbx) {
    using G = L1Geom<float, TH, TW>;
    constexpr int PH = TH / 2, PW = TW / 2, CNT = PH * PW;
    double acc[NSUM] = {0, 0, 0, 0, 0};
    static_for<0, 4>([&](auto cp) {
        constexpr int P = decltype(cp)::value >> 1, Q = decltype(cp)::value & 1;
        float loc[NSUM] = {0.f, 0.f, 0.f, 0.f, 0.f};
        // unrolled: the global loads (u_prev, f) of all the thread's pixels of the
        // plane are issued before their first use (a rolled loop pays one memory
        // latency per pixel)
#pragma unroll
        for (int itr = 0; itr < (CNT + NTH - 1) / NTH; ++itr) {
            const int t = threadIdx.x + itr * NTH;
            if (t >= CNT) continue;
            const int ii = t / PW, kk = t % PW;
            const int gi = R + 2 * ii + P, gk = C + 2 * kk + Q;
            if (gi >= m || gk >= n) continue;
            const QuadAcc<float, TH, TW, P, Q> A{su, G::HALO / 2 + ii, G::HALO / 2 + kk};
            const float c = A.template at<0, 0>();
            const long long g = (long long)gi * n + gk;
            const float fv = FG ? __ldg(f + g)
                                : sf[(P * 2 + Q) * G::PLANE + (G::HALO / 2 + ii) * G::QW + G::HALO / 2 + kk];
            loc[0] += curv_term<float>(c, A.template at<0, 1>(), A.template at<0, -1>(), A.template at<-1, 0>(),
                                       A.template at<1, 0>(), A.template at<-1, 1>(), A.template at<1, -1>(),
                                       A.template at<-1, -1>(), A.template at<1, 1>(), MODE_MEAN);
            const float d = c - fv;
            loc[1] += d * d;
            loc[2] += fabsf(c - __ldg(up + g));
            loc[3] += fabsf(c);
            if (rf) {
                const float dr = c - __ldg(rf + g);
                loc[4] += dr * dr;
            }
        }
#pragma unroll
        for (int s2 = 0; s2 < NSUM; ++s2) acc[s2] += (double)loc[s2];
    });
    cta_sums_store(acc, partials, nbx, cta, b);
}

// FG: f is not staged in shared memory but read from global memory (L2) by
// the pixel's own phase: half the shared memory per CTA, more CTAs per SM
template <int TH, int TW, int NR, bool FAST = true, int NT = 256, bool FG = false, bool EF = false>
__global__ void __launch_bounds__(NT) k_l1_x2(FusedArgs<float> a) {
    pdl_sync();
    using G = L1Geom<float, TH, TW>;
    static_assert(G::QW % 2 == 0, "pairs must stay 8-byte aligned");
    constexpr int PAIRS = G::QW / 2;             // packed pairs per plane row
    constexpr int ROWS_PER_PASS = NT / PAIRS;    // plane rows handled per pass
    static_assert(NT % PAIRS == 0, "");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* su = reinterpret_cast<float*>(smem_raw) + 2;  // 2 guard words: p[-1] at the first pair stays in bounds
    float* sf = su + 4 * G::PLANE;
    const int b = blockIdx.z;
    const int R = blockIdx.y * TH, C = blockIdx.x * TW;
    const float* uin = a.uin + (long long)b * a.istride;
    const float* f = a.f + (long long)b * a.istride;
    float* uout = a.uout + (long long)b * a.istride;
    const int m = a.m, n = a.n;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x, nbx = gridDim.x * gridDim.y;
    if (a.st[b].done) {  // stopped image (final u in ImgState::final_buf)
        if constexpr (EF) efused_ticket(a.fz, a.partials, nbx, b, reinterpret_cast<double*>(smem_raw));
        return;
    }
    const int r0 = R - G::HALO, c0 = C - G::HALO;
    const bool border = (r0 < 1) || (c0 < 1) || (r0 + G::RH >= m) || (c0 + G::RW >= n);
    const bool vec = !border && (n % 4 == 0);
    if (vec) {
        // 16-byte loads: 4 consecutive pixels -> two 8-byte pairs of the two column planes.
        // Thread t owns float4 column c4 = t % V4 of region rows t / V4 + j * RSTEP: one 64-bit
        // base pointer, constant row strides, a fixed row parity (RSTEP is even) and
        // compile-time shared-memory offsets.
        constexpr int V4 = G::RW / 4;
        constexpr int RSTEP = NT / V4;
        constexpr int NV4 = (G::RH + RSTEP - 1) / RSTEP;
        static_assert(NT % V4 == 0 && RSTEP % 2 == 0, "staging map");
        const int c4 = threadIdx.x % V4, row = threadIdx.x / V4;
        const long long g0 = (long long)(r0 + row) * n + c0 + 4 * c4;
        const float4* ub = reinterpret_cast<const float4*>(uin + g0);
        const float4* fbp = reinterpret_cast<const float4*>(f + g0);
        const int rstride4 = RSTEP * (n / 4);  // float4 per RSTEP image rows
        {
            // L2 prefetch of every 128-byte line of the region (u and f) first: the
            // register-staged loads below then merge into requests already in flight
            constexpr int LPR = G::RW / 32 + 1;  // lines per region row (c0 is not line aligned)
            constexpr int NPF = 2 * G::RH * LPR;
            for (int e = threadIdx.x; e < NPF && !(a.dbg & 0x10000); e += NT) {  // CMG_DBG bit 16: off
                const int arr = e / (G::RH * LPR), rem = e % (G::RH * LPR);
                const float* base = (arr ? f : uin) + (long long)(r0 + rem / LPR) * n + c0 + 32 * (rem % LPR);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base));
            }
        }
        float4 uv[NV4], fv4[NV4];
#pragma unroll
        for (int j = 0; j < NV4; ++j) {
            if (G::RH % RSTEP == 0 || row + j * RSTEP < G::RH) {
                uv[j] = __ldg(ub + j * rstride4);
                if constexpr (!FG) fv4[j] = __ldg(fbp + j * rstride4);
            }
        }
        const int s0 = (row & 1) * 2 * G::PLANE + (row >> 1) * G::QW + 2 * c4;  // plane (p,0), word 2*c4
#pragma unroll
        for (int j = 0; j < NV4; ++j) {
            if (G::RH % RSTEP == 0 || row + j * RSTEP < G::RH) {
                const int o = s0 + j * (RSTEP / 2) * G::QW;
                *reinterpret_cast<unsigned long long*>(su + o) = f2_pack(uv[j].x, uv[j].z).v;
                *reinterpret_cast<unsigned long long*>(su + o + G::PLANE) = f2_pack(uv[j].y, uv[j].w).v;
                if constexpr (!FG) {
                    *reinterpret_cast<unsigned long long*>(sf + o) = f2_pack(fv4[j].x, fv4[j].z).v;
                    *reinterpret_cast<unsigned long long*>(sf + o + G::PLANE) = f2_pack(fv4[j].y, fv4[j].w).v;
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < G::RH * G::RW; e += blockDim.x) {
            const int i = e / G::RW, k = e % G::RW;
            const int gi = r0 + i, gk = c0 + k;
            if (gi >= 0 && gi < m && gk >= 0 && gk < n) {
                const long long g = (long long)gi * n + gk;
                su[G::idx(i, k)] = uin[g];
                if constexpr (!FG) sf[G::idx(i, k)] = f[g];
            }
        }
    }
    __syncthreads();
    if (border) l1_reflect_fix<float, TH, TW>(su, r0, c0, m, n);
    if constexpr (EF)
        x2_energy_sums<TH, TW, FG, NT>(su, sf, f, R, C, m, n, a.uprev + (long long)b * a.istride,
                                   a.ref ? a.ref + (long long)b * a.istride : nullptr, a.partials, b, cta, nbx);
    const F2 w2 = f2_splat((float)a.P->w[1][0]);
    const F2 inv2 = f2_splat((float)(1.0 / a.P->den[1][0]));
    const F2 nz2 = f2_splat(a.nz);  // -0.0f (see mul2)
    F2 finite_acc = f2_splat(0.f);  // stays 0 unless a correction is inf/NaN (x*0)
    const F2 zero2 = f2_splat(0.f);
    const int prow = threadIdx.x / PAIRS, pj = threadIdx.x % PAIRS;
    if (!border && FAST) {
        // Interior tile: a thread owns pair column pj and plane rows prow + k*ROWS_PER_PASS in every
        // phase, so all neighbour addresses are one base register + a compile-time offset and the only
        // per-pair bookkeeping is the phase's row / column range.
        constexpr int ITERS = (G::QH + ROWS_PER_PASS - 1) / ROWS_PER_PASS;
        const float* sb = su + prow * G::QW + 2 * pj;
        float* sbw = su + prow * G::QW + 2 * pj;
        const float* fb = sf + prow * G::QW + 2 * pj;
        static_for<0, 4>([&](auto cphase) {
            constexpr int c = decltype(cphase)::value;
            constexpr int P = c >> 1, Q = c & 1;
            constexpr int h = 3 - c;
            constexpr int i_min = G::HALO - h, i_max = G::HALO + TH + h;
            constexpr int k_min = G::HALO - h, k_max = G::HALO + TW + h;
            constexpr int qi_lo = (i_min - P + 1) / 2, qi_hi = (i_max - P + 1) / 2;
            constexpr int PL_c = (P * 2 + Q) * G::PLANE;
            constexpr int PL_ns = ((1 - P) * 2 + Q) * G::PLANE;
            constexpr int PL_ew = (P * 2 + (1 - Q)) * G::PLANE;
            constexpr int PL_d = ((1 - P) * 2 + (1 - Q)) * G::PLANE;
            constexpr int aN = (P - 1) >> 1, aS = (P + 1) >> 1;
            constexpr int bE = (Q + 1) >> 1;
            const int kA = 4 * pj + Q;
            const bool okA = kA >= k_min && kA < k_max, okB = kA + 2 >= k_min && kA + 2 < k_max;
            static_for<0, ITERS>([&](auto itc) {
                constexpr int it = decltype(itc)::value;
                constexpr int OFF = it * ROWS_PER_PASS * G::QW;
                const int qi = prow + it * ROWS_PER_PASS;
                if (qi >= qi_lo && qi < qi_hi && (okA || okB)) {
                    auto pairEW = [&](auto rowoff, auto plane, F2& Ev, F2& Wv) {
                        const float* p = sb + (decltype(plane)::value + OFF + decltype(rowoff)::value * G::QW);
                        const F2 al = lds2(p);
                        float lo, hi;
                        f2_unpack(al, lo, hi);
                        if constexpr (bE == 0) {
                            Ev = al;
                            Wv = f2_pack(p[-1], lo);
                        } else {
                            Wv = al;
                            Ev = f2_pack(hi, p[2]);
                        }
                    };
                    using IC0 = std::integral_constant<int, 0>;
                    using ICN = std::integral_constant<int, aN>;
                    using ICS = std::integral_constant<int, aS>;
                    using ICEW = std::integral_constant<int, PL_ew>;
                    using ICD = std::integral_constant<int, PL_d>;
                    const F2 cv = lds2(sb + (PL_c + OFF));
                    F2 fv;
                    if constexpr (FG) {  // pixels (i, 4pj+Q) and (i, 4pj+Q+2) of the region
                        const float* fp = f + (long long)(r0 + 2 * qi + P) * n + c0 + 4 * pj + Q;
                        fv = f2_pack(__ldg(fp), __ldg(fp + 2));
                    } else {
                        fv = lds2(fb + (PL_c + OFF));
                    }
                    const F2 Nv = lds2(sb + (PL_ns + OFF + aN * G::QW));
                    const F2 Sv = lds2(sb + (PL_ns + OFF + aS * G::QW));
                    F2 Ev, Wv, NEv, NWv, SEv, SWv;
                    pairEW(IC0{}, ICEW{}, Ev, Wv);
                    pairEW(ICN{}, ICD{}, NEv, NWv);
                    pairEW(ICS{}, ICD{}, SEv, SWv);
                    const F2 ch = l1_chalf_x2<NR>(cv, Ev, Wv, Nv, Sv, NEv, NWv, SEv, SWv, nz2);
                    const F2 corr = mul2(fma2(w2, fv - cv, ch), inv2, nz2);
                    F2 nu = cv + corr;
                    if (!(okA && okB)) {
                        float c0v, c1v, n0, n1;
                        f2_unpack(cv, c0v, c1v);
                        f2_unpack(nu, n0, n1);
                        nu = f2_pack(okA ? n0 : c0v, okB ? n1 : c1v);
                    }
                    *reinterpret_cast<unsigned long long*>(sbw + (PL_c + OFF)) = nu.v;
                }
            });
            __syncthreads();
        });
        // non-finite corrections: every pixel's final value is computed identically by the tile
        // that owns it, and a non-finite correction leaves a non-finite value -> check the outputs
    } else
    static_for<0, 4>([&](auto cphase) {
        constexpr int c = decltype(cphase)::value;
        constexpr int P = c >> 1, Q = c & 1;
        constexpr int h = 3 - c;
        // valid region rows/cols of this colour phase: [HALO-h, HALO+T+h)
        constexpr int i_min = G::HALO - h, i_max = G::HALO + TH + h;  // half-open
        constexpr int k_min = G::HALO - h, k_max = G::HALO + TW + h;
        constexpr int qi_lo = (i_min - P + 1) / 2, qi_hi = (i_max - P + 1) / 2;  // 2qi+P in [i_min,i_max)
        // plane offsets of the neighbours: plane (rp,cq), row shift a, col shift b
        constexpr int PL_c = (P * 2 + Q) * G::PLANE;
        constexpr int PL_ns = ((1 - P) * 2 + Q) * G::PLANE;          // N and S live in the other row parity
        constexpr int PL_ew = (P * 2 + (1 - Q)) * G::PLANE;          // E and W
        constexpr int PL_d = ((1 - P) * 2 + (1 - Q)) * G::PLANE;     // diagonals
        constexpr int aN = (P - 1) >> 1, aS = (P + 1) >> 1;          // row shift of N / S
        constexpr int bW = (Q - 1) >> 1, bE = (Q + 1) >> 1;          // col shift of W / E (one of them is 0)
        for (int qi = qi_lo + prow; qi < qi_hi; qi += ROWS_PER_PASS) {
            const int qk = 2 * pj;
            const int base = qi * G::QW + qk;
            // aligned pairs (b = 0) and the one extra scalar for the b = +-1 side
            auto pairEW = [&](int rowoff, int plane, F2& Ev, F2& Wv) {
                const float* p = su + plane + base + rowoff * G::QW;
                const F2 al = lds2(p);  // columns qk, qk+1 of that plane
                float lo, hi;
                f2_unpack(al, lo, hi);
                if constexpr (bE == 0) {  // E aligned, W = (p[-1], lo)
                    Ev = al;
                    Wv = f2_pack(p[-1], lo);
                } else {  // W aligned, E = (hi, p[2])
                    Wv = al;
                    Ev = f2_pack(hi, p[2]);
                }
            };
            const F2 cv = lds2(su + PL_c + base);
            F2 fv;
            if constexpr (FG) {  // clamped: out-of-image pixels are discarded below
                const int gi = min(max(r0 + 2 * qi + P, 0), m - 1);
                const int ga = min(max(c0 + 4 * pj + Q, 0), n - 1), gb = min(max(c0 + 4 * pj + Q + 2, 0), n - 1);
                fv = f2_pack(__ldg(f + (long long)gi * n + ga), __ldg(f + (long long)gi * n + gb));
            } else {
                fv = lds2(sf + PL_c + base);
            }
            const F2 Nv = lds2(su + PL_ns + base + aN * G::QW);
            const F2 Sv = lds2(su + PL_ns + base + aS * G::QW);
            F2 Ev, Wv, NEv, NWv, SEv, SWv;
            pairEW(0, PL_ew, Ev, Wv);
            pairEW(aN, PL_d, NEv, NWv);
            pairEW(aS, PL_d, SEv, SWv);
            const F2 ch = l1_chalf_x2<NR>(cv, Ev, Wv, Nv, Sv, NEv, NWv, SEv, SWv, nz2);
            const F2 corr = mul2(fma2(w2, fv - cv, ch), inv2, nz2);  // (c_half + w f*) / (2 + w), f* = f - u
            F2 nu = cv + corr;
            float c0v, c1v, n0, n1, k0, k1;
            f2_unpack(cv, c0v, c1v);
            f2_unpack(nu, n0, n1);
            f2_unpack(corr, k0, k1);
            // validity of the two pixels: phase column range and (border tiles) the image
            const int i = 2 * qi + P;
            const int kA = 2 * qk + Q, kB = kA + 2;
            bool okA = kA >= k_min && kA < k_max, okB = kB >= k_min && kB < k_max;
            if (border) {
                const int gi = r0 + i;
                const bool rin = gi >= 0 && gi < m;
                okA = okA && rin && (c0 + kA) >= 0 && (c0 + kA) < n;
                okB = okB && rin && (c0 + kB) >= 0 && (c0 + kB) < n;
            }
            finite_acc = fma2(f2_pack(okA ? k0 : 0.f, okB ? k1 : 0.f), zero2, finite_acc);
            nu = f2_pack(okA ? n0 : c0v, okB ? n1 : c1v);
            *reinterpret_cast<unsigned long long*>(su + PL_c + base) = nu.v;
        }
        __syncthreads();
        if (border) l1_reflect_fix<float, TH, TW>(su, r0, c0, m, n);
    });
    const bool vec_out = (R + TH <= m) && (C + TW <= n) && (n % 4 == 0);
    if (vec_out) {
        // thread t writes float4 column c4 = t % CW (< TW/4) of tile rows t / CW + j * OSTEP
        constexpr int TV4 = TW / 4;
        constexpr int CW = TV4 <= 8 ? 8 : (TV4 <= 16 ? 16 : 32);
        constexpr int OSTEP = NT / CW;
        constexpr int NO = (TH + OSTEP - 1) / OSTEP;
        static_assert(NT % CW == 0 && OSTEP % 2 == 0 && TV4 <= 32, "output map");
        const int c4 = threadIdx.x % CW, row = threadIdx.x / CW;
        if (c4 < TV4) {
            float4* op = reinterpret_cast<float4*>(uout + (long long)(R + row) * n + C + 4 * c4);
            const int ostride4 = OSTEP * (n / 4);
            // region pixel (HALO + row, HALO + 4 c4): row parity fixed, even column -> word HALO/2 + 2 c4
            const int s0 = ((G::HALO + row) & 1) * 2 * G::PLANE + ((G::HALO + row) >> 1) * G::QW + G::HALO / 2 + 2 * c4;
#pragma unroll
            for (int j = 0; j < NO; ++j) {
                if (TH % OSTEP == 0 || row + j * OSTEP < TH) {
                    const int o = s0 + j * (OSTEP / 2) * G::QW;
                    const F2 v02 = lds2(su + o), v13 = lds2(su + o + G::PLANE);
                    if (!border && FAST) finite_acc = fma2(v13, zero2, fma2(v02, zero2, finite_acc));
                    float x0, x2, x1, x3;
                    f2_unpack(v02, x0, x2);
                    f2_unpack(v13, x1, x3);
                    op[j * ostride4] = make_float4(x0, x1, x2, x3);
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < TH * TW; e += blockDim.x) {
            const int i = e / TW, k = e % TW;
            const int gi = R + i, gk = C + k;
            if (gi < m && gk < n) {
                const float v = su[G::idx(i + G::HALO, k + G::HALO)];
                if (!border && FAST) finite_acc = fma2(f2_pack(v, 0.f), zero2, finite_acc);
                uout[(long long)gi * n + gk] = v;
            }
        }
    }
    float fa0, fa1;
    f2_unpack(finite_acc, fa0, fa1);
    const bool bad = !(isfinite(fa0) && isfinite(fa1));
    if (__syncthreads_or(bad) && threadIdx.x == 0) {
        if constexpr (EF) {
            a.st[b].bad1 = 1;
            __threadfence();  // visible to the CTA that finalizes (efused_ticket)
        } else {
            a.st[b].bad = 1;
        }
    }
    if constexpr (EF) {
        __syncthreads();  // shared memory becomes the finalize scratch
        efused_ticket(a.fz, a.partials, nbx, b, reinterpret_cast<double*>(smem_raw));
    }
}

}  // namespace cmg
