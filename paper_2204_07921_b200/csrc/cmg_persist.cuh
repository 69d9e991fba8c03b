// cmg_persist.cuh -- the whole denoise (driver.denoise, driver.py:261-314) as
// ONE persistent cooperative kernel.
//
// Each colour sweep of each level is a grid-wide phase separated by a grid
// barrier; the energy phase also refreshes u_prev, and every CTA reduces the
// energy partials itself (same fixed order in every CTA) so all CTAs reach the
// same stopping decision without a second barrier.  Phases per V-cycle:
// 4*J colour sweeps + 1 energy = 13 barriers for J=3, zero kernel launches.
//
// Used for every image that does not need numpy's iterated reflection (the
// padded-snapshot path stays on the multi-kernel graph).
#pragma once

#include <cooperative_groups.h>

#include "cmg_kernels.cuh"

namespace cmg {

namespace cg = cooperative_groups;

struct PersistArgs {
    void* u;
    void* uprev;
    const void* f;
    const void* ref;
    long long N;  // pixels per image
    int m, n, B;
    int nseq;
    int seq[12];
    int hc[7][4], wc[7][4], side[7];
    const SolveParams* P;
    ImgState* st;
    TraceArgs tr;
    double* partials;  // [B][npieces][NSUM]
    int npieces;
    long long piece;
    int has_ref;
};

template <typename T>
__device__ __forceinline__ SweepArgs<T> make_sweep_args(const PersistArgs& a, int layer, int color) {
    SweepArgs<T> s;
    s.u = (T*)a.u;
    s.f = (const T*)a.f;
    s.istride = a.N;
    s.upad = nullptr;
    s.fpad = nullptr;
    s.pstride = 0;
    s.W = 0;
    s.m = a.m;
    s.n = a.n;
    s.layer = layer;
    s.s = a.side[layer];
    s.r = 1 << (layer - 1);
    s.p = color >> 1;
    s.q = color & 1;
    s.hc = a.hc[layer][color];
    s.wc = a.wc[layer][color];
    s.flat = (s.wc == 1);
    s.single = (s.hc * s.wc == 1);
    s.P = a.P;
    s.st = a.st;
    s.dbg = 0;
    s.bk.inner = a.P->inner;
    s.bk.w0 = a.P->w[layer][0];
    s.bk.den0 = a.P->den[layer][0];
    s.bk.inv0 = 1.0 / s.bk.den0;
    return s;
}

// level 1: one thread per patch (pixel), grid-stride
template <typename T, int MODE, int PREC>
__device__ __forceinline__ void phase_level1(const SweepArgs<T>& s, int B, const int* sdone) {
    const long long per = (long long)s.hc * s.wc;
    const long long total = per * B;
    const long long gth = (long long)gridDim.x * blockDim.x;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gth) {
        const int b = (int)(g / per);
        if (sdone[b]) continue;
        const long long r = g - (long long)b * per;
        const int pr = (int)(r / s.wc), pc = (int)(r % s.wc);
        const int R0 = 2 * pr + s.p, C0 = 2 * pc + s.q;
        T* u = s.u + (long long)b * s.istride;
        const T* f = s.f + (long long)b * s.istride;
        T c;
        if ((R0 >= 1) && (C0 >= 1) && (R0 + 1 < s.m) && (C0 + 1 < s.n)) {
            Direct<T> U{u, s.n}, F{f, s.n};
            c = patch_solve_ct<T, 1, MODE, PREC>(U, F, R0, C0, s);
        } else {
            c = patch_solve_ct_border<T, 1, MODE, PREC>(u, f, R0, C0, s);
        }
        if (!isfinite(c)) s.st[b].bad = 1;
        T* p = u + (long long)R0 * s.n + C0;
        *p = X<T>::add(*p, c);
    }
}

// levels 2-3: TS lanes per patch, grid-stride over teams (warp-uniform trip count)
template <typename T, int LAYER, int MODE, int PREC, int TS>
__device__ __forceinline__ void phase_team(const SweepArgs<T>& s, int B, const int* sdone) {
    constexpr int S = (1 << LAYER) - 1;
    const long long per = (long long)s.hc * s.wc;
    const long long total = per * B;
    const long long nteams = (long long)gridDim.x * (blockDim.x / TS);
    const long long team = (long long)blockIdx.x * (blockDim.x / TS) + threadIdx.x / TS;
    const int lane = threadIdx.x % TS;
    const long long iters = (total + nteams - 1) / nteams;
    for (long long it = 0; it < iters; ++it) {
        long long idx = team + it * nteams;
        bool valid = idx < total;
        if (!valid) idx = total - 1;
        const int b = (int)(idx / per);
        if (sdone[b]) valid = false;
        const long long r = idx - (long long)b * per;
        const int pr = (int)(r / s.wc), pc = (int)(r % s.wc);
        const int R0 = (2 * pr + s.p) * S, C0 = (2 * pc + s.q) * S;
        T* u = s.u + (long long)b * s.istride;
        const T* f = s.f + (long long)b * s.istride;
        T c;
        const bool inside = (R0 >= 1) && (C0 >= 1) && (R0 + S < s.m) && (C0 + S < s.n);
        if (__all_sync(0xffffffffu, inside)) {
            Direct<T> U{u, s.n}, F{f, s.n};
            c = patch_solve_team<T, LAYER, MODE, PREC, TS>(U, F, R0, C0, lane, s);
        } else {
            c = patch_solve_team_border<T, LAYER, MODE, PREC, TS>(u, f, R0, C0, lane, s);
        }
        // every lane of every team of this warp has consumed its reads (the
        // shuffles above are warp-synchronous), so the writes may start
        if (valid) {
            if (lane == 0 && !isfinite(c)) s.st[b].bad = 1;
            for (int e = lane; e < S * S; e += TS) {
                const int i = R0 + e / S, k = C0 + e % S;
                if (i < s.m && k < s.n) {
                    T* p = u + (long long)i * s.n + k;
                    *p = X<T>::add(*p, c);
                }
            }
        }
    }
}

// levels 4-6: one CTA per patch, grid-stride over patches
template <typename T, int MODE>
__device__ __forceinline__ void phase_bpp(const SweepArgs<T>& s, int B, const int* sdone, T* sh_rows, T* sh_vals,
                                          T* sh_c) {
    const int S = s.s;
    const long long per = (long long)s.hc * s.wc;
    const long long total = per * B;
    for (long long idx = blockIdx.x; idx < total; idx += gridDim.x) {
        const int b = (int)(idx / per);
        if (sdone[b]) continue;  // block-uniform
        const long long r = idx - (long long)b * per;
        const int pr = (int)(r / s.wc), pc = (int)(r % s.wc);
        const int R0 = (2 * pr + s.p) * S, C0 = (2 * pc + s.q) * S;
        T* u = s.u + (long long)b * s.istride;
        const T* f = s.f + (long long)b * s.istride;
        if ((R0 >= 1) && (C0 >= 1) && (R0 + S < s.m) && (C0 + S < s.n)) {
            Direct<T> U{u, s.n}, F{f, s.n};
            bpp_body<T, MODE>(U, F, R0, C0, s, sh_rows, sh_vals, sh_c);
        } else {
            Reflect<T> U{u, s.m, s.n}, F{f, s.m, s.n};
            bpp_body<T, MODE>(U, F, R0, C0, s, sh_rows, sh_vals, sh_c);
        }
        __syncthreads();
        const T c = *sh_c;
        if (threadIdx.x == 0 && !isfinite(c)) s.st[b].bad = 1;
        const int r1 = min(R0 + S, s.m), c1 = min(C0 + S, s.n);
        const int w = c1 - C0, h = r1 - R0;
        for (int e = threadIdx.x; e < w * h; e += blockDim.x) {
            T* p = u + (long long)(R0 + e / w) * s.n + (C0 + e % w);
            *p = X<T>::add(*p, c);
        }
        __syncthreads();
    }
}

// energy partial sums per (image, piece); also u_prev <- u for the next cycle
template <typename T>
__device__ __forceinline__ void phase_energy(const PersistArgs& a, int mode, const int* sdone, double* sh_red) {
    const long long items = (long long)a.B * a.npieces;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int b = (int)(it / a.npieces);
        const int pcx = (int)(it % a.npieces);
        double acc[NSUM] = {0, 0, 0, 0, 0};
        if (!sdone[b]) {
            const T* u = (const T*)a.u + (long long)b * a.N;
            const T* f = (const T*)a.f + (long long)b * a.N;
            T* up = (T*)a.uprev + (long long)b * a.N;
            const T* rf = a.has_ref ? (const T*)a.ref + (long long)b * a.N : nullptr;
            const long long e0 = (long long)pcx * a.piece;
            const long long e1 = min(a.N, e0 + a.piece);
            for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
                const int i = (int)(e / a.n), k = (int)(e % a.n);
                double uo, uE, uW, uN, uS, uNE, uSW, uNW, uSE;
                auto ld = [&](const auto& A) {
                    uo = (double)A(i, k);
                    uE = (double)A(i, k + 1);
                    uW = (double)A(i, k - 1);
                    uN = (double)A(i - 1, k);
                    uS = (double)A(i + 1, k);
                    uNE = (double)A(i - 1, k + 1);
                    uSW = (double)A(i + 1, k - 1);
                    uNW = (double)A(i - 1, k - 1);
                    uSE = (double)A(i + 1, k + 1);
                };
                if (i >= 1 && k >= 1 && i + 1 < a.m && k + 1 < a.n)
                    ld(Direct<T>{u, a.n});
                else
                    ld(Reflect<T>{u, a.m, a.n});
                const double two = 2.0 * uo;
                const double k0 = ((uE + uW) - two) * 0.5;
                const double k1 = ((uN + uS) - two) * 0.5;
                const double k2 = ((uNE + uSW) - two) * 0.25;
                const double k3 = ((uNW + uSE) - two) * 0.25;
                const double kmin = fmin(fmin(k0, k1), fmin(k2, k3));
                const double kmax = fmax(fmax(k0, k1), fmax(k2, k3));
                double term = (mode == MODE_MEAN) ? fabs(0.5 * (kmin + kmax)) : fabs(kmin * kmax);
                if (isnan(k0) || isnan(k1) || isnan(k2) || isnan(k3)) term = __longlong_as_double(0x7ff8000000000000ULL);
                const T uT = u[e];
                const double uv = (double)uT;
                const double d = uv - (double)f[e];
                acc[0] += term;
                acc[1] += d * d;
                acc[2] += fabs(uv - (double)up[e]);
                acc[3] += fabs(uv);
                if (rf) {
                    const double dr = uv - (double)rf[e];
                    acc[4] += dr * dr;
                }
                up[e] = uT;
            }
        }
        // deterministic block reduction -> partials[b][pcx]
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
        for (int s = 0; s < NSUM; ++s) {
            double v = acc[s];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) sh_red[s * 32 + wid] = v;
        }
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
#pragma unroll
            for (int s = 0; s < NSUM; ++s) {
                double v = lane < nw ? sh_red[s * 32 + lane] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                if (lane == 0) a.partials[((long long)b * a.npieces + pcx) * NSUM + s] = v;
            }
        }
        __syncthreads();
    }
}

// Every CTA reduces every running image's partials in the same order and
// applies the stopping rule to its shared copy of the state; CTA 0 also
// writes the trace and the global state.  Returns nothing; updates sdone/sF.
__device__ __forceinline__ void phase_finalize(const PersistArgs& a, int initial, int cycle, int* sdone, double* sF,
                                               unsigned long long t0) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const SolveParams* P = a.P;
    for (int b = wid; b < a.B; b += nw) {
        if (sdone[b]) continue;  // warp-uniform
        double acc[NSUM] = {0, 0, 0, 0, 0};
        for (int i = lane; i < a.npieces; i += 32)
#pragma unroll
            for (int s = 0; s < NSUM; ++s) acc[s] += a.partials[((long long)b * a.npieces + i) * NSUM + s];
#pragma unroll
        for (int s = 0; s < NSUM; ++s)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], o);
        if (lane != 0) continue;
        const double F = acc[0] + P->half_alpha * acc[1];
        const double du = acc[2], au = acc[3], dr = acc[4];
        const bool writer = (blockIdx.x == 0);
        const long long base = (long long)b * a.tr.cap;
        double ps = __longlong_as_double(0x7ff8000000000000ULL);
        if (P->has_ref) {
            const double mse = dr / (double)P->npix;
            ps = (mse == 0.0) ? __longlong_as_double(0x7ff0000000000000ULL) : 10.0 * log10(P->peak * P->peak / mse);
        }
        ImgState& S = a.st[b];
        if (initial) {
            sF[b] = F;
            if (writer) {
                S.F = F;
                S.cycle = 0;
                S.done = 0;
                S.status = ST_RUNNING;
                S.t0 = t0;
                a.tr.energy[base] = F;
                a.tr.rel_e[base] = __longlong_as_double(0x7ff8000000000000ULL);
                a.tr.rel_u[base] = __longlong_as_double(0x7ff8000000000000ULL);
                a.tr.psnr[base] = ps;
                a.tr.seconds[base] = 0.0;
            }
            continue;
        }
        int status = ST_RUNNING;
        if (S.bad) {
            status = ST_NONFINITE;
        } else if (!isfinite(F)) {
            status = ST_DIVERGED;
            if (writer) a.tr.energy[base + cycle] = F;
        } else {
            const double Fo = sF[b];
            const double re = (F == 0.0) ? fabs(Fo) : fabs(F - Fo) / fabs(F);
            const double ru =
                (au == 0.0) ? ((du == 0.0) ? 0.0 : __longlong_as_double(0x7ff0000000000000ULL)) : du / au;
            sF[b] = F;
            if (writer) {
                a.tr.energy[base + cycle] = F;
                a.tr.rel_e[base + cycle] = re;
                a.tr.rel_u[base + cycle] = ru;
                a.tr.psnr[base + cycle] = ps;
                a.tr.seconds[base + cycle] = (double)(globaltimer() - t0) * 1e-9;
                S.F = F;
                S.cycle = cycle;
            }
            const double crit = (P->stop_rule == 0) ? re : ru;
            if (crit <= P->eps)
                status = ST_CONVERGED;
            else if (cycle >= P->max_outer)
                status = ST_NOT_CONVERGED;
        }
        if (status != ST_RUNNING) {
            sdone[b] = 1;
            if (writer) {
                S.status = status;
                S.done = 1;
                atomicAdd(a.tr.ndone, 1);
            }
        }
    }
}

template <typename T, int MODE, int PREC, int TS2, int TS3>
__global__ void __launch_bounds__(256) k_persist(PersistArgs a) {
    pdl_sync();
    extern __shared__ __align__(16) unsigned char smem[];
    double* sF = reinterpret_cast<double*>(smem);
    int* sdone = reinterpret_cast<int*>(sF + a.B);
    double* sh_red = reinterpret_cast<double*>(sdone + ((a.B + 1) & ~1));
    T* sh_rows = reinterpret_cast<T*>(sh_red + NSUM * 32);
    T* sh_vals = sh_rows + 64;
    T* sh_c = sh_vals + 256;
    cg::grid_group grid = cg::this_grid();
    const unsigned long long t0 = globaltimer();

    for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
        sdone[b] = 0;
        sF[b] = 0.0;
    }
    // u = f, u_prev = f   (driver.py:277)
    {
        const long long tot = a.N * a.B;
        const T* f = (const T*)a.f;
        T* u = (T*)a.u;
        T* up = (T*)a.uprev;
        for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
             e += (long long)gridDim.x * blockDim.x) {
            const T v = f[e];
            u[e] = v;
            up[e] = v;
        }
    }
    __syncthreads();
    grid.sync();
    phase_energy<T>(a, MODE, sdone, sh_red);
    grid.sync();
    phase_finalize(a, 1, 0, sdone, sF, t0);
    __syncthreads();

    for (int cycle = 1;; ++cycle) {
        for (int si = 0; si < a.nseq; ++si) {
            const int j = a.seq[si];
            for (int c = 0; c < 4; ++c) {
                if (a.hc[j][c] <= 0 || a.wc[j][c] <= 0) continue;
                const SweepArgs<T> s = make_sweep_args<T>(a, j, c);
                if (j == 1)
                    phase_level1<T, MODE, PREC>(s, a.B, sdone);
                else if (j == 2)
                    phase_team<T, 2, MODE, PREC, TS2>(s, a.B, sdone);
                else if (j == 3)
                    phase_team<T, 3, MODE, PREC, TS3>(s, a.B, sdone);
                else
                    phase_bpp<T, MODE>(s, a.B, sdone, sh_rows, sh_vals, sh_c);
                grid.sync();
            }
        }
        phase_energy<T>(a, MODE, sdone, sh_red);
        grid.sync();
        phase_finalize(a, 0, cycle, sdone, sF, t0);
        __syncthreads();
        int running = 0;
        for (int b = threadIdx.x; b < a.B; b += blockDim.x) running |= !sdone[b];
        if (!__syncthreads_or(running)) break;
    }
}

}  // namespace cmg

namespace cmg {

// Levels >= 2 of one V-cycle segment (e.g. [2, 3]) as ONE cooperative kernel:
// each colour of each level is a grid-wide phase (team-per-patch, in place on
// a.u) separated by grid barriers -- replaces 4 launches per level when the
// image is small enough that a colour sweep is latency-bound.
template <typename T, int MODE, int PREC, int TS2, int TS3>
__global__ void __launch_bounds__(256) k_coarse_coop(PersistArgs a) {
    pdl_sync();
    extern __shared__ __align__(16) unsigned char smem[];
    int* sdone = reinterpret_cast<int*>(smem);
    T* sh_rows = reinterpret_cast<T*>(smem + 16 * ((a.B * sizeof(int) + 15) / 16));
    T* sh_vals = sh_rows + 64;
    T* sh_c = sh_vals + 256;
    cg::grid_group grid = cg::this_grid();
    for (int b = threadIdx.x; b < a.B; b += blockDim.x) sdone[b] = a.st[b].done;
    __syncthreads();
    bool first = true;
    for (int si = 0; si < a.nseq; ++si) {
        const int j = a.seq[si];
        for (int c = 0; c < 4; ++c) {
            if (a.hc[j][c] <= 0 || a.wc[j][c] <= 0) continue;
            if (!first) grid.sync();
            first = false;
            const SweepArgs<T> s = make_sweep_args<T>(a, j, c);
            if (j == 2)
                phase_team<T, 2, MODE, PREC, TS2>(s, a.B, sdone);
            else if (j == 3)
                phase_team<T, 3, MODE, PREC, TS3>(s, a.B, sdone);
            else
                phase_bpp<T, MODE>(s, a.B, sdone, sh_rows, sh_vals, sh_c);
        }
    }
}

}  // namespace cmg
