// cmg_rowpair.cuh -- levels 2-3 as two launches per level visit: one per
// patch-row parity p, each running the colours (p,0) then (p,1)
// (driver.sweep_layer, driver.py:225-251, COLOR_ORDER driver.py:35).
//
// Why this split is exact.  The stencil of a patch reaches one pixel beyond
// it, so a colour-(p,1) patch reads the (p,0) patches to its
// left and right and the patch rows above and below, which have the other
// parity and are not modified by either colour of this launch.  A CTA owns a
// patch row and TPC consecutive patch columns; it stages the rows
// [R0-1, R0+S] of its window (owned patches, one read-only patch on the left,
// one (p,0) halo patch on the right) in shared memory, runs colour (p,0),
// refreshes the odd-reflection cells, runs colour (p,1) and writes its owned
// pixels.  The halo patch is computed redundantly (bit-identical to its
// owner's result).
//
// Buffers: the level reads X and writes Y (the fused-level rotation).  The
// p=0 launch reads everything from X and writes the parity-0 patch rows of Y;
// the p=1 launch reads its own rows from X and the parity-0 rows (its ring
// rows, and mirror rows of the bottom reflection) from Y, where they are
// final.  No CTA ever reads a pixel another CTA of the same launch writes.
//
// Compared with four in-place colour launches this halves the launches and
// the HBM traffic of a level (each launch reads (S+2)/2S of u and half of f
// and writes half of u).
#pragma once

#include "cmg_kernels.cuh"
#include "cmg_coarse.cuh"

namespace cmg {

template <typename T>
struct RowPairArgs {
    const T* X;      // level input (u before this level)
    T* Y;            // level output
    int ntiles;      // column tiles per patch row
    int nj;          // patch columns
    SweepArgs<T> c0, c1;  // colours (p,0) and (p,1): p, q, hc, wc, flat, single, backward constants
};

// shared-memory window accessor in padded image coordinates
template <typename T>
struct WinAcc {
    const T* s;
    int ld, r0, k0;
    __device__ __forceinline__ T operator()(int i, int k) const { return s[(i - r0) * ld + (k - k0)]; }
};

// TPC_ > 0: fewer owned patch columns than the teams could take (an even count that
// covers a narrow image in one tile: 64 x 512^2 at level 3 has 74 patch columns)
template <int LAYER, int TS, int NT_ = 256, int A_ = 1, int TPC_ = 0>
struct RowPairGeom {
    static constexpr int S = (1 << LAYER) - 1;
    static constexpr int NT = NT_;
    static constexpr int TEAMS = NT / TS;
    static constexpr int TPC = TPC_ > 0 ? TPC_ : 2 * TEAMS - 2;  // owned patch columns per CTA (even)
    static_assert(TPC % 2 == 0 && TPC <= 2 * TEAMS - 2, "owned patch columns");
    // window columns: [(J0-1)S-1, (J0+TPC+1)S]; with A_ > 1 the window origin is
    // floored to a multiple of A_ elements (16-byte aligned bulk copies) and the
    // width padded to a multiple of A_ that still covers the shifted window
    static constexpr int WIN0 = (TPC + 2) * S + 2;
    static constexpr int WIN = A_ == 1 ? WIN0 : ((WIN0 + 2 * (A_ - 1)) / A_) * A_;
    static constexpr int ROWS = S + 2;                 // window rows: [R0-1, R0+S]
};

// one work item: patch row PR of image b, owned patch columns [J0, J0+TPC)
template <typename T>
struct RPItem {
    int b, R0, J0, wr0, wk0, orow1, ok0, ok1;
    bool border;
    const T *Xb, *f;
    T* Yb;
};

template <typename T, int LAYER, int TS, int NT, int TPC_ = 0>
__device__ __forceinline__ RPItem<T> rp_item(const RowPairArgs<T>& a, int b, int pr, int tile) {
    using G = RowPairGeom<LAYER, TS, NT, 1, TPC_>;
    constexpr int S = G::S;
    const SweepArgs<T>& A0 = a.c0;
    const int m = A0.m, n = A0.n;
    RPItem<T> it;
    it.b = b;
    it.R0 = (2 * pr + A0.p) * S;
    it.J0 = tile * G::TPC;
    it.wr0 = it.R0 - 1;
    it.wk0 = (it.J0 - 1) * S - 1;  // window origin (padded coordinates)
    // owned pixels: rows [R0, min(R0+S, m)), columns [J0 S, min((J0+TPC) S, n))
    it.orow1 = min(it.R0 + S, m);
    it.ok0 = it.J0 * S;
    it.ok1 = min((it.J0 + G::TPC) * S, n);
    it.border = (it.wr0 < 0) || (it.wr0 + G::ROWS > m) || (it.wk0 < 0) || (it.wk0 + G::WIN > n);
    const long long ioff = (long long)b * A0.istride;
    it.Xb = a.X + ioff;
    it.Yb = a.Y + ioff;
    it.f = A0.f + ioff;
    return it;
}

// pixels of parity-0 patch rows are final in Y during the p=1 launch
template <typename T, int S>
__device__ __forceinline__ const T* rp_src_row(const RPItem<T>& it, int p, int i) {
    return (p == 1 && ((i / S) & 1) == 0) ? it.Yb : it.Xb;
}

// stage the in-image cells of an item's window: u rows R0-1 .. R0+S into win,
// f rows R0 .. R0+S-1 into fwin = win + ROWS*WIN.
template <typename T, int LAYER, int TS, int NT>
__device__ __forceinline__ void rp_stage(const RowPairArgs<T>& a, const RPItem<T>& it, T* win) {
    using G = RowPairGeom<LAYER, TS, NT>;
    constexpr int S = G::S;
    const int m = a.c0.m, n = a.c0.n, p = a.c0.p;
    T* fwin = win + G::ROWS * G::WIN;
    const int wlo = max(it.wk0, 0), whi = min(it.wk0 + G::WIN, n);  // in-image window columns
    // per column: every row's load is issued before the first shared-memory store
    // (one global round trip per column instead of one per row)
    constexpr int NR = G::ROWS + S;  // u rows R0-1 .. R0+S, then f rows R0 .. R0+S-1
    const T* srow[G::ROWS];
#pragma unroll
    for (int ri = 0; ri < G::ROWS; ++ri) {
        const int i = it.wr0 + ri;
        srow[ri] = rp_src_row<T, S>(it, p, i) + (long long)i * n;
    }
    const T* frow0 = it.f + (long long)it.R0 * n;
    const int nr = a.c0.fsum ? G::ROWS : NR;  // fast mean with per-patch f sums: no f pixels needed
    for (int k = wlo + threadIdx.x; k < whi; k += G::NT) {
        T v[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int i = (r < G::ROWS) ? it.wr0 + r : it.R0 + (r - G::ROWS);
            if (r < nr && i >= 0 && i < m)
                v[r] = (r < G::ROWS) ? srow[r][k] : __ldg(frow0 + (long long)(r - G::ROWS) * n + k);
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int i = (r < G::ROWS) ? it.wr0 + r : it.R0 + (r - G::ROWS);
            if (r < nr && i >= 0 && i < m) {
                if (r < G::ROWS)
                    win[r * G::WIN + (k - it.wk0)] = v[r];
                else
                    fwin[(r - G::ROWS) * G::WIN + (k - it.wk0)] = v[r];
            }
        }
    }
}

// everything after staging: border refills, the two colours, write-back.
// Starts and ends with the window consistent across the CTA (callers sync
// before; this ends with a barrier-free write-back of owned pixels).
// EDGES_ONLY: the caller bulk-stores the A-aligned interior of each owned row;
// the threads write only the (< A) unaligned columns at both ends
template <typename T, int LAYER, int MODE, int PREC, int TS, int NT, int A = 1, bool EDGES_ONLY = false,
          int TPC_ = 0>
__device__ __forceinline__ void rp_compute(const RowPairArgs<T>& a, const RPItem<T>& it, T* win) {
    using G = RowPairGeom<LAYER, TS, NT, A, TPC_>;
    constexpr int S = G::S;
    const SweepArgs<T>& A0 = a.c0;
    const int m = A0.m, n = A0.n, p = A0.p;
    const int R0 = it.R0, J0 = it.J0, wr0 = it.wr0, wk0 = it.wk0;
    T* fwin = win + G::ROWS * G::WIN;
    const int wlo = max(wk0, 0), whi = min(wk0 + G::WIN, n);
    const int kmax = A0.W - 2;  // np (padded columns run -1 .. np)
    if (it.border && !A0.fsum) {  // padded f cells of the patch row (f is constant: reflect from global)
        const Reflect<T> FR{it.f, m, n};
        for (int e = threadIdx.x; e < S * G::WIN; e += G::NT) {
            const int ri = e / G::WIN, ck = e % G::WIN;
            const int i = R0 + ri, k = wk0 + ck;
            if ((i >= m || k == -1 || k >= n) && k >= -1 && k <= kmax) fwin[ri * G::WIN + ck] = FR(i, k);
        }
    }
    // odd reflection (rows first, then columns: tangent.py:262-269) of the window's
    // out-of-image u cells within one pixel of the padded image; in-image sources come
    // from the window when inside it, else from the level's stable rows in global memory
    auto refill = [&]() {
        auto g = [&](int i, int k) -> T {
            const int ri = i - wr0, ck = k - wk0;
            if (ri >= 0 && ri < G::ROWS && ck >= 0 && ck < G::WIN) return win[ri * G::WIN + ck];
            return rp_src_row<T, S>(it, p, i)[(long long)i * n + k];
        };
        auto rowv = [&](int i, int k) -> T {
            if (i >= 0 && i < m) return g(i, k);
            const int e = (i < 0) ? 0 : m - 1;
            const int mi = (i < 0) ? -i : 2 * (m - 1) - i;
            return X<T>::sub(X<T>::mul(T(2), g(e, k)), g(mi, k));
        };
        for (int ri = 0; ri < G::ROWS; ++ri) {  // rows beyond the image, in-image columns
            const int i = wr0 + ri;
            if (i >= 0 && i < m) continue;
            for (int k = wlo + threadIdx.x; k < whi; k += G::NT) win[ri * G::WIN + (k - wk0)] = rowv(i, k);
        }
        __syncthreads();
        // columns beyond the image (column -1 and n .. np): reflect the row-padded values
        const int klo = max(wk0, n), khi = min(wk0 + G::WIN - 1, kmax);
        for (int ri = threadIdx.x / 32; ri < G::ROWS; ri += G::NT / 32) {
            const int i = wr0 + ri;
            for (int k = klo + (threadIdx.x & 31); k <= khi; k += 32)
                win[ri * G::WIN + (k - wk0)] =
                    X<T>::sub(X<T>::mul(T(2), rowv(i, n - 1)), rowv(i, 2 * (n - 1) - k));
            if (wk0 <= -1 && (threadIdx.x & 31) == 0)
                win[ri * G::WIN + (-1 - wk0)] = X<T>::sub(X<T>::mul(T(2), rowv(i, 0)), rowv(i, 1));
        }
        __syncthreads();
    };
    if (it.border) refill();
    const WinAcc<T> U{win, G::WIN, wr0, wk0};
    const WinAcc<T> F{fwin, G::WIN, R0, wk0};
    const int lane = threadIdx.x % TS, team = threadIdx.x / TS;
    bool bad = false;
    // the two colours of this patch row: (p,0) on J0, J0+2, ..., J0+TPC (the last one
    // is the halo the (p,1) patch J0+TPC-1 needs), then (p,1) on J0+1, ..., J0+TPC-1
    static_for<0, 2>([&](auto qc) {
        constexpr int q = decltype(qc)::value;
        const SweepArgs<T>& A = q ? a.c1 : a.c0;
        const int J = J0 + q + 2 * team;
        const bool active = (J < a.nj) && (q == 0 ? J <= J0 + G::TPC : J < J0 + G::TPC) && A.wc > 0;
        if (__any_sync(0xffffffffu, active)) {
            const int Jc = active ? J : J0;  // inactive teams shadow a valid patch (converged shuffles)
            const int C0 = Jc * S;
            const double* fsp =
                A.fsum ? A.fsum + (long long)it.b * A.fs_img + (long long)(R0 / S) * A.fs_ld + Jc : nullptr;
            const T c = patch_solve_team<T, LAYER, MODE, PREC, TS>(U, F, R0, C0, lane, A, fsp);
            if (active) {
                if (lane == 0 && !isfinite(c)) bad = true;
                // prolongation u += c on the patch's in-image pixels (hierarchy.py:117-126);
                // the element loop has a compile-time trip count (e / S, e % S fold for TS = 1)
                T* base = win + (R0 - wr0) * G::WIN + (C0 - wk0);
                const int rmax = min(S, m - R0), cmax = min(S, n - C0);
#pragma unroll
                for (int t = 0; t < (S * S + TS - 1) / TS; ++t) {
                    const int e = lane + t * TS;
                    const int r = e / S, k = e - (e / S) * S;
                    if (e < S * S && r < rmax && k < cmax) {
                        T* px = base + r * G::WIN + k;
                        *px = X<T>::add(*px, c);
                    }
                }
            }
        }
        // the caller's bulk stores (async proxy) read what these threads wrote
        if constexpr (EDGES_ONLY && q == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (q == 0 && it.border) refill();
    });
    if (bad) A0.st[it.b].bad = 1;
    // owned pixels -> Y
    if constexpr (EDGES_ONLY) {
        const int a0 = min(((it.ok0 + A - 1) / A) * A, it.ok1), a1 = max((it.ok1 / A) * A, a0);
        const int nl = a0 - it.ok0, ne = nl + (it.ok1 - a1);
        const int rows = it.orow1 - R0;
        for (int e = threadIdx.x; e < rows * ne; e += G::NT) {
            const int i = R0 + e / ne, j = e % ne;
            const int k = j < nl ? it.ok0 + j : a1 + (j - nl);
            it.Yb[(long long)i * n + k] = win[(i - wr0) * G::WIN + (k - wk0)];
        }
    } else {
        for (int i = R0; i < it.orow1; ++i)
            for (int k = it.ok0 + threadIdx.x; k < it.ok1; k += G::NT)
                it.Yb[(long long)i * n + k] = win[(i - wr0) * G::WIN + (k - wk0)];
    }
}

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <typename T, int LAYER, int MODE, int PREC, int TS, int NT = 256>
__global__ void __launch_bounds__(NT) k_rowpair(RowPairArgs<T> a) {
    pdl_sync();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* win = reinterpret_cast<T*>(smem_raw);
    const RPItem<T> it = rp_item<T, LAYER, TS, NT>(a, blockIdx.z, blockIdx.y, blockIdx.x);
    if (a.c0.st[it.b].done) return;  // stopped image (final u in ImgState::final_buf)
    rp_stage<T, LAYER, TS, NT>(a, it, win);
    __syncthreads();
    rp_compute<T, LAYER, MODE, PREC, TS, NT>(a, it, win);
}

// ---------------------------------------------------------------------------
// k_rowpair with bulk-copy staging (latency-bound jobs: config 3's levels 2-3).
// One item per CTA as in k_rowpair, but the window rows (u rows R0-1 .. R0+S,
// then the f rows R0 .. R0+S-1) arrive by one cp.async.bulk each, issued by
// the lanes of warp 0 and completed on one mbarrier, and the A-aligned
// interior of the owned rows leaves by bulk stores: the per-column staging and
// write-back loops (40 % of k_rowpair's instructions at level 3) disappear.
// The window origin is floored to A = 16/sizeof(T) columns so shared-memory
// and global columns share their 16-byte phase.  Requires n*sizeof(T) % 16 == 0.
// ---------------------------------------------------------------------------
template <typename T, int LAYER, int MODE, int PREC, int TS, int NT = 256>
__global__ void __launch_bounds__(NT) k_rowpair_tma(RowPairArgs<T> a) {
    pdl_sync();
    if (a.c0.dbg & 8) return;  // diagnostics: launch cost only
    constexpr int A = 16 / (int)sizeof(T);
    using G = RowPairGeom<LAYER, TS, NT, A>;
    constexpr int S = G::S;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* win = reinterpret_cast<T*>(smem_raw);
    __shared__ __align__(8) unsigned long long full;
    const int m = a.c0.m, n = a.c0.n, p = a.c0.p;
    RPItem<T> it = rp_item<T, LAYER, TS, NT>(a, blockIdx.z, blockIdx.y, blockIdx.x);
    it.wk0 = (it.wk0 >= 0) ? (it.wk0 / A) * A : -(((-it.wk0) + A - 1) / A) * A;
    it.border = (it.wr0 < 0) || (it.wr0 + G::ROWS > m) || (it.wk0 < 0) || (it.wk0 + G::WIN > n);
    const bool fs = a.c0.fsum != nullptr;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int wlo = max(it.wk0, 0), whi = min(it.wk0 + G::WIN, n);
        const unsigned bytes = (unsigned)(whi - wlo) * (unsigned)sizeof(T);
        // lane r < ROWS: u row wr0 + r; ROWS <= r < ROWS + S: f row R0 + r - ROWS
        const int nr = G::ROWS + (fs ? 0 : S);
        const int i = lane < G::ROWS ? it.wr0 + lane : it.R0 + (lane - G::ROWS);
        const bool valid = lane < nr && i >= 0 && i < m;
        const unsigned cnt = __popc(__ballot_sync(0xffffffffu, valid));
        if (lane == 0) {
            mbar_init(&full, 1);
            mbar_expect_tx(&full, bytes * cnt);
        }
        __syncwarp();
        if (valid) {
            const T* src = lane < G::ROWS ? rp_src_row<T, S>(it, p, i) : it.f;
            bulk_g2s(win + lane * G::WIN + (wlo - it.wk0), src + (long long)i * n + wlo, bytes, &full);
        }
    }
    const bool done = a.c0.st[it.b].done != 0;
    __syncthreads();  // barrier initialised
    mbar_wait(&full, 0u);
    if (done) return;  // stopped image (final u in ImgState::final_buf); the copies have landed
    if (a.c0.dbg & 16) return;  // diagnostics: launch + staging
    rp_compute<T, LAYER, MODE, PREC, TS, NT, A, true>(a, it, win);
    if (threadIdx.x == 0) {
        const int a0 = min(((it.ok0 + A - 1) / A) * A, it.ok1), a1 = max((it.ok1 / A) * A, a0);
        if (a1 > a0) {
            for (int i = it.R0; i < it.orow1; ++i)
                bulk_s2g(it.Yb + (long long)i * n + a0, win + (i - it.wr0) * G::WIN + (a0 - it.wk0),
                         (unsigned)(a1 - a0) * (unsigned)sizeof(T));
            bulk_commit();
            bulk_wait_read0();  // shared memory stays valid until the stores have read it
        }
    }
}

// ---------------------------------------------------------------------------
// Large jobs, fast mean mode with per-patch f sums: the same row-parity
// launches, one thread per patch, as a PERSISTENT kernel whose windows are
// streamed by bulk asynchronous copies (cp.async.bulk + mbarrier, one copy per
// window row) into two shared-memory stages: item i+1's rows are in flight
// while item i computes.  u only (no f pixels).  Requires n*sizeof(T) % 16 == 0.
// ---------------------------------------------------------------------------
template <typename T, int LAYER, int NT, int STAGES, int TPC_ = 0>
__global__ void __launch_bounds__(NT) k_rowpair_bulk(RowPairArgs<T> a, int rows, int B) {
    pdl_sync();
    constexpr int A = 16 / (int)sizeof(T);
    using G = RowPairGeom<LAYER, 1, NT, A, TPC_>;
    constexpr int STAGE = G::ROWS * G::WIN;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stage0 = reinterpret_cast<T*>(smem_raw);
    __shared__ __align__(8) unsigned long long full[STAGES];
    const int tid = threadIdx.x;
    const int m = a.c0.m, n = a.c0.n, p = a.c0.p;
    const long long per_img = (long long)rows * a.ntiles;
    const long long items = per_img * B;
    auto item_of = [&](long long itx) {
        const int b = (int)(itx / per_img);
        const long long r = itx - (long long)b * per_img;
        const int pr = (int)(r / a.ntiles), tile = (int)(r - (long long)pr * a.ntiles);
        RPItem<T> x = rp_item<T, LAYER, 1, NT, TPC_>(a, b, pr, tile);
        x.wk0 = (x.wk0 >= 0) ? (x.wk0 / A) * A : -(((-x.wk0) + A - 1) / A) * A;
        x.border = (x.wr0 < 0) || (x.wr0 + G::ROWS > m) || (x.wk0 < 0) || (x.wk0 + G::WIN > n);
        return x;
    };
    // thread 0: one bulk copy per in-image window row (16-byte aligned ends);
    // the stage's pending bulk stores must have read it first
    auto issue = [&](const RPItem<T>& x, T* win, unsigned long long* bar) {
        bulk_wait_read0();
        if (a.c0.st[x.b].done) {
            mbar_expect_tx(bar, 0u);
            return;
        }
        const int wlo = max(x.wk0, 0), whi = min(x.wk0 + G::WIN, n);
        const unsigned bytes = (unsigned)(whi - wlo) * (unsigned)sizeof(T);
        int nrow = 0;
#pragma unroll
        for (int ri = 0; ri < G::ROWS; ++ri) {
            const int i = x.wr0 + ri;
            nrow += (i >= 0 && i < m) ? 1 : 0;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes of the previous item
        mbar_expect_tx(bar, bytes * (unsigned)nrow);
#pragma unroll
        for (int ri = 0; ri < G::ROWS; ++ri) {
            const int i = x.wr0 + ri;
            if (i >= 0 && i < m)
                bulk_g2s(win + ri * G::WIN + (wlo - x.wk0), rp_src_row<T, G::S>(x, p, i) + (long long)i * n + wlo, bytes,
                         bar);
        }
    };
    // thread 0: bulk stores of the A-aligned interior of the owned rows (the
    // threads wrote the unaligned ends); smem column k and global column k share
    // their 16-byte phase because the window origin is A-aligned
    auto store = [&](const RPItem<T>& x, const T* win) {
        const int a0 = min(((x.ok0 + A - 1) / A) * A, x.ok1), a1 = max((x.ok1 / A) * A, a0);
        if (a1 <= a0) return;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = x.R0; i < x.orow1; ++i)
            bulk_s2g(x.Yb + (long long)i * n + a0, win + (i - x.wr0) * G::WIN + (a0 - x.wk0),
                     (unsigned)(a1 - a0) * (unsigned)sizeof(T));
        bulk_commit();
    };
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    __syncthreads();
    long long itx = blockIdx.x;
    if (STAGES > 1 && tid == 0 && itx < items) issue(item_of(itx), stage0, &full[0]);
    for (int i = 0; itx < items; itx += gridDim.x, ++i) {
        const RPItem<T> cur = item_of(itx);
        const int st = i % STAGES;
        if (tid == 0) {
            if (STAGES == 1) {
                issue(cur, stage0, &full[0]);
            } else {
                const long long nx = itx + gridDim.x;
                if (nx < items) issue(item_of(nx), stage0 + ((i + 1) % STAGES) * STAGE, &full[(i + 1) % STAGES]);
            }
        }
        mbar_wait(&full[st], (unsigned)((i / STAGES) & 1));
        T* win = stage0 + st * STAGE;
        if (!a.c0.st[cur.b].done) {
            rp_compute<T, LAYER, MODE_MEAN, PREC_FAST, 1, NT, A, true, TPC_>(a, cur, win);
            if (tid == 0) store(cur, win);
        }
        __syncthreads();  // the stage is refilled by a later iteration's copy
    }
    if (tid == 0) bulk_wait0();
}

}  // namespace cmg
