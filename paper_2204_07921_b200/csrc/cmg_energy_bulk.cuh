// cmg_energy_bulk.cuh -- energy + finalize with rows streamed into shared
// memory by bulk asynchronous copies (cp.async.bulk + mbarrier ring).
//
// The energy pass reads u (3x3 neighbourhood), f, u_prev and ref once per
// pixel: an HBM-bound stream with almost no arithmetic.  Register-staged
// loads keep too few bytes in flight (the row-band kernel reaches ~2.3 TB/s
// at 16384^2), so here one thread per CTA streams whole row segments through
// an NS-deep ring of shared-memory stages while the 256 threads consume them:
// NS x ~16 KB in flight per CTA, independent of register pressure.
//
// Work item = band of H rows x CW = 256*PX columns (PX pixels = 16 bytes per
// thread).  Step t of an item (t = -2 .. H-1) brings u row i0+t+1 (with a
// 16-byte halo on each side) and, for t >= 0, row i0+t of f / u_prev / ref.
// Each thread keeps the 3 x (PX+2) window of u in registers, exactly as the
// row-band kernel.  Sums: the PX terms of a thread's row segment are added in
// the image precision in a fixed order, then to fp64 accumulators.
// Requires n * sizeof(T) % 16 == 0 (16-byte aligned rows).
#pragma once

#include "cmg_coarse.cuh"
#include "cmg_kernels.cuh"

namespace cmg {

template <typename T, int PX>
struct EBGeom {
    static constexpr int CW = 256 * PX;                 // columns per item
    static constexpr int PADL = 16 / (int)sizeof(T);    // halo elements each side (16 bytes)
    static constexpr int UW = CW + 2 * PADL;            // u row segment
    static constexpr int SLOT = UW + 3 * CW;            // u | f | u_prev | ref (16-byte multiple)
    static constexpr int MAXNS = 8;
};

// out-of-image u row (i = -1 or m): odd reflection from global memory (rare)
template <typename T, int PX>
static __device__ __noinline__ void eb_row_reflect(const T* u, int m, int n, int i, int k0, T* v) {
    Reflect<T> R{u, m, n};
#pragma unroll
    for (int j = 0; j < PX + 2; ++j) v[j] = R(i, k0 - 1 + j);
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// PX consecutive elements from shared memory as one 4/8/16-byte access
template <typename T, int PX>
__device__ __forceinline__ void eb_lds(const T* p, T (&v)[PX]) {
    constexpr int BYTES = PX * (int)sizeof(T);
    if constexpr (BYTES == 16) {
        const uint4 w = *reinterpret_cast<const uint4*>(p);
        const T* q = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int j = 0; j < PX; ++j) v[j] = q[j];
    } else if constexpr (BYTES == 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        const T* q = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int j = 0; j < PX; ++j) v[j] = q[j];
    } else {
#pragma unroll
        for (int j = 0; j < PX; ++j) v[j] = p[j];
    }
}

// 8 consumer warps (256 threads, PX pixels each) + 1 producer warp whose lane
// 0 issues the bulk copies.  Ring of NS stages: full[s] completes when the
// stage's bytes have landed, empty[s] when all 8 consumer warps released it.
template <typename T, int PX>
__global__ void __launch_bounds__(288) k_energy_bulk(EnergyArgs a, EnergyFin fz, int H, int NS) {
    pdl_sync();
    using G = EBGeom<T, PX>;
    using A = T;
    extern __shared__ __align__(128) unsigned char eb_smem[];
    T* slots = reinterpret_cast<T*>(eb_smem);
    __shared__ __align__(8) unsigned long long full[G::MAXNS], empty[G::MAXNS];
    const int b = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31;
    double acc[NSUM] = {0, 0, 0, 0, 0};
    if (!a.st[b].done) {  // uniform per CTA
        const T* u = (const T*)a.u + (long long)b * a.istride;
        const int n = a.n, m = a.m;
        const int r_lo = (int)(a.e_lo / n), r_hi = (int)(a.e_hi / n);
        const int nrb = (r_hi - r_lo + H - 1) / H, ncb = (n + G::CW - 1) / G::CW;
        const long long items = (long long)nrb * ncb;
        const bool has_ref = a.ref != nullptr;
        if (tid == 0)
            for (int s = 0; s < NS; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 8);
            }
        __syncthreads();
        if (tid >= 256) {
            // ---------------- producer ----------------
            if (lane == 0) {
                const T* f = (const T*)a.f + (long long)b * a.istride;
                const T* up = (const T*)a.uprev + (long long)b * a.istride;
                const T* rf = has_ref ? (const T*)a.ref + (long long)b * a.istride : nullptr;
                int slot = 0, fills = 0;
                unsigned epar = 0;
                for (long long it = blockIdx.x; it < items; it += a.nbx) {
                    const int rb = (int)(it / ncb), cb = (int)(it - (long long)rb * ncb);
                    const int i0 = r_lo + rb * H, i1 = min(r_hi, i0 + H);
                    const int c0 = cb * G::CW;
                    const int lo = max(c0 - G::PADL, 0), hi = min(c0 + G::CW + G::PADL, n);
                    const int fw = min(c0 + G::CW, n) - c0;
                    const unsigned ub = (unsigned)(hi - lo) * sizeof(T), fb = (unsigned)fw * sizeof(T);
                    for (int t = -2; t < i1 - i0; ++t) {
                        if (fills >= NS) mbar_wait(&empty[slot], epar);
                        T* su = slots + slot * G::SLOT;
                        const int r = i0 + t + 1;
                        const bool rin = r >= 0 && r < m;
                        mbar_expect_tx(&full[slot], (rin ? ub : 0u) + (t >= 0 ? fb * (has_ref ? 3u : 2u) : 0u));
                        if (rin) bulk_g2s(su + (lo - (c0 - G::PADL)), u + (long long)r * n + lo, ub, &full[slot]);
                        if (t >= 0) {
                            const long long e = (long long)(i0 + t) * n + c0;
                            bulk_g2s(su + G::UW, f + e, fb, &full[slot]);
                            bulk_g2s(su + G::UW + G::CW, up + e, fb, &full[slot]);
                            if (has_ref) bulk_g2s(su + G::UW + 2 * G::CW, rf + e, fb, &full[slot]);
                        }
                        ++fills;
                        if (++slot == NS) {
                            slot = 0;
                            if (fills > NS) epar ^= 1u;
                        }
                    }
                }
            }
        } else {
            // ---------------- consumers ----------------
            int slot = 0;
            unsigned fpar = 0;
            const int sb = tid * PX + G::PADL;  // smem index of the thread's first column in a u segment
            for (long long it = blockIdx.x; it < items; it += a.nbx) {
                const int rb = (int)(it / ncb), cb = (int)(it - (long long)rb * ncb);
                const int i0 = r_lo + rb * H, i1 = min(r_hi, i0 + H);
                const int k0 = cb * G::CW + tid * PX;
                const bool kin = k0 < n;
                const bool eL = k0 == 0, eR = k0 + PX == n;
                A N[PX + 2], C[PX + 2];
                for (int t = -2; t < i1 - i0; ++t) {
                    mbar_wait(&full[slot], fpar);
                    const T* su = slots + slot * G::SLOT;
                    const int r = i0 + t + 1;
                    A S[PX + 2];
                    if (r >= 0 && r < m) {  // uniform
                        T c[PX];
                        eb_lds<T, PX>(su + sb, c);
#pragma unroll
                        for (int j = 0; j < PX; ++j) S[j + 1] = c[j];
                        const T lft = __shfl_up_sync(0xffffffffu, c[PX - 1], 1);
                        const T rgt = __shfl_down_sync(0xffffffffu, c[0], 1);
                        S[0] = lane == 0 ? su[sb - 1] : lft;
                        S[PX + 1] = lane == 31 ? su[sb + PX] : rgt;
                        // odd reflection at the image edges (as Reflect)
                        if (eL) S[0] = X<T>::sub(X<T>::mul(T(2), S[1]), S[2]);
                        if (eR) S[PX + 1] = X<T>::sub(X<T>::mul(T(2), S[PX]), S[PX - 1]);
                    } else if (kin) {
                        T tmp[PX + 2];
                        eb_row_reflect<T, PX>(u, m, n, r, k0, tmp);
#pragma unroll
                        for (int j = 0; j < PX + 2; ++j) S[j] = tmp[j];
                    }
                    if (t >= 0 && kin) {
                        const T* sf = su + G::UW + tid * PX;
                        T fv[PX], pv[PX], rv[PX];
                        eb_lds<T, PX>(sf, fv);
                        eb_lds<T, PX>(sf + G::CW, pv);
                        if (has_ref) {
                            eb_lds<T, PX>(sf + 2 * G::CW, rv);
                        } else {
#pragma unroll
                            for (int j = 0; j < PX; ++j) rv[j] = T(0);
                        }
                        // the PX (<= 4) terms of a thread's row segment are added in the image
                        // precision, then accumulated in fp64: for fp32 a 4-term group adds at
                        // most ~3 ulp of relative error, the size of the fp32 per-pixel terms
                        // themselves (the per-row / 8-row chunks of k_energy are fp64 per pixel)
                        A tv[NSUM][PX];
#pragma unroll
                        for (int j = 0; j < PX; ++j) {
                            const A cc = C[j + 1];
                            tv[0][j] = curv_term<A>(cc, C[j + 2], C[j], N[j + 1], S[j + 1], N[j + 2], S[j], N[j],
                                                    S[j + 2], a.mode);
                            const A d = cc - fv[j];
                            tv[1][j] = d * d;
                            tv[2][j] = fabs(cc - pv[j]);
                            tv[3][j] = fabs(cc);
                            const A dr = cc - rv[j];
                            tv[4][j] = has_ref ? dr * dr : A(0);
                        }
#pragma unroll
                        for (int s = 0; s < NSUM - 1; ++s) {
                            A v = tv[s][0];
                            if (PX == 2) v = tv[s][0] + tv[s][1];
                            if (PX == 4) v = (tv[s][0] + tv[s][1]) + (tv[s][2] + tv[s][3]);
                            acc[s] += (double)v;
                        }
                        if (has_ref) {  // (u - ref)^2 only with a reference image
                            constexpr int s = NSUM - 1;
                            A v = tv[s][0];
                            if (PX == 2) v = tv[s][0] + tv[s][1];
                            if (PX == 4) v = (tv[s][0] + tv[s][1]) + (tv[s][2] + tv[s][3]);
                            acc[s] += (double)v;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < PX + 2; ++j) {
                        N[j] = C[j];
                        C[j] = S[j];
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[slot]);
                    if (++slot == NS) {
                        slot = 0;
                        fpar ^= 1u;
                    }
                }
            }
        }
    }
    energy_reduce_finalize(acc, a, fz, b);
}

template <typename T, int PX>
constexpr size_t eb_smem_bytes(int NS) {
    return (size_t)NS * EBGeom<T, PX>::SLOT * sizeof(T);
}

}  // namespace cmg
