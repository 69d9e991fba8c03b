// cmg_launch.cuh -- kernel launch sequences per element type (instantiated in
// cmg_f64.cu / cmg_f32.cu so the two dtypes compile in parallel).
#pragma once

#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "cmg_fused.cuh"
#include "cmg_l1.cuh"
#include "cmg_l1x2.cuh"
#include "cmg_l1loop.cuh"
#include "cmg_coarse.cuh"
#include "cmg_energy_bulk.cuh"
#include "cmg_rowpair.cuh"
#include "cmg_plan.h"

namespace cmg {

template <typename T>
void enqueue_pad(cmg_plan* P, const void* src, void* dst, int H, int W, long long pstride, int bot, int rgt,
                 bool gate) {
    const ImgState* st = gate ? P->st : nullptr;
    const int blocks = (int)std::min<long long>((P->N + 255) / 256, 4096);
    klaunch(P, k_pad_copy<T>, dim3(blocks, P->B), 256, 0, (const T*)src, P->N, (T*)dst, pstride, P->m, P->n, W,
                                                             st);
    klaunch(P, k_pad_axis<T>, dim3((P->n + 127) / 128, P->B), 128, 0, (T*)dst, pstride, 0, P->m, P->n, H, W,
                                                                         bot, rgt, st);
    klaunch(P, k_pad_axis<T>, dim3((H + 127) / 128, P->B), 128, 0, (T*)dst, pstride, 1, P->m, P->n, H, W, bot,
                                                                      rgt, st);
    P->enq += 3;
}

template <typename T, int LAYER, int MODE, int PREC>
void launch_tpp(const cmg_plan* P, const SweepArgs<T>& a, bool padded, int B) {
    const dim3 blk(32, 8);
    const dim3 grd((a.wc + 31) / 32, (a.hc + 7) / 8, B);
    if (padded)
        klaunch(P, k_sweep_tpp<T, LAYER, MODE, PREC, SRC_PADDED>, grd, blk, 0, a);
    else
        klaunch(P, k_sweep_tpp<T, LAYER, MODE, PREC, SRC_INPLACE>, grd, blk, 0, a);
}

template <typename T, int LAYER, int MODE, int PREC, int TS>
void launch_team(const cmg_plan* P, const SweepArgs<T>& a, bool padded, int B) {
    const long long np = (long long)a.hc * a.wc;
    const int per_block = 256 / TS;
    const dim3 grd((unsigned)((np + per_block - 1) / per_block), 1, B);
    if (padded)
        klaunch(P, k_sweep_team<T, LAYER, MODE, PREC, SRC_PADDED, TS>, grd, 256, 0, a);
    else
        klaunch(P, k_sweep_team<T, LAYER, MODE, PREC, SRC_INPLACE, TS>, grd, 256, 0, a);
}

template <typename T, int MODE, int PREC>
void dispatch_small_layer(const cmg_plan* P, const SweepArgs<T>& a, bool padded) {
    switch (a.layer) {
        case 1: launch_tpp<T, 1, MODE, PREC>(P, a, padded, P->B); break;
        case 2:
            if (P->ts2 == 16)
                launch_team<T, 2, MODE, PREC, 16>(P, a, padded, P->B);
            else if (P->ts2 == 8)
                launch_team<T, 2, MODE, PREC, 8>(P, a, padded, P->B);
            else
                launch_team<T, 2, MODE, PREC, 4>(P, a, padded, P->B);
            break;
        default:
            if (P->ts3 == 32)
                launch_team<T, 3, MODE, PREC, 32>(P, a, padded, P->B);
            else if (P->ts3 == 16)
                launch_team<T, 3, MODE, PREC, 16>(P, a, padded, P->B);
            else
                launch_team<T, 3, MODE, PREC, 8>(P, a, padded, P->B);
            break;
    }
}

// kernel arguments of one colour of a level (driver.sweep_layer, driver.py:225-251)
template <typename T>
SweepArgs<T> make_sweep_args(const cmg_plan* P, int layer, int color) {
    const Level& L = P->lv[layer];
    const int p = color >> 1, q = color & 1;
    const int hc = (L.mj - p + 1) / 2, wc = (L.nj - q + 1) / 2;
    SweepArgs<T> a;
    a.u = (T*)P->u;
    a.f = (const T*)P->f;
    a.istride = P->N;
    a.upad = (const T*)P->upad;
    a.fpad = (const T*)L.fpad;
    a.pstride = L.pstride;
    a.W = L.W;
    a.m = P->m;
    a.n = P->n;
    a.layer = layer;
    a.s = L.s;
    a.r = L.r;
    a.p = p;
    a.q = q;
    a.hc = hc;
    a.wc = wc;
    a.flat = (wc == 1);      // NumPy coalesces a single patch column
    a.single = (hc * wc == 1);  // single patch: d.mean(axis=0) becomes pairwise
    a.P = P->P;
    a.st = P->st;
    a.dbg = P->dbg;
    a.bk.inner = P->hostP.inner;
    a.bk.w0 = P->hostP.w[layer][0];
    a.bk.den0 = P->hostP.den[layer][0];
    a.bk.inv0 = 1.0 / P->hostP.den[layer][0];
    a.fsum = (layer <= 3) ? P->fsum[layer] : nullptr;
    a.fs_img = (long long)L.mj * L.nj;
    a.fs_ld = L.nj;
    return a;
}

// per-patch f sums of levels 2-3 (fast mean mode): after every change of f
template <typename T>
void enqueue_fsums(cmg_plan* P) {
    for (int j = 2; j <= std::min(P->layers, 3); ++j) {
        if (!P->fsum[j]) continue;
        const Level& L = P->lv[j];
        const long long np = (long long)L.mj * ((L.nj + 3) / 4);  // one thread per group of four patches
        const dim3 grd((unsigned)((np + 255) / 256), P->B);
        if (j == 2)
            klaunch(P, k_patch_fsum<T, 3>, grd, 256, 0, (const T*)P->f, P->fsum[j], P->m, P->n, L.mj, L.nj, P->N);
        else
            klaunch(P, k_patch_fsum<T, 7>, grd, 256, 0, (const T*)P->f, P->fsum[j], P->m, P->n, L.mj, L.nj, P->N);
        P->enq += 1;
    }
}

template <typename T>
void enqueue_sweep(cmg_plan* P, int layer, int color) {
    Level& L = P->lv[layer];
    const int p = color >> 1, q = color & 1;
    const int hc = (L.mj - p + 1) / 2, wc = (L.nj - q + 1) / 2;
    if (hc <= 0 || wc <= 0) return;
    if (L.general) enqueue_pad<T>(P, P->u, P->upad, L.H, L.W, L.pstride, 1 + L.mp - P->m, 1 + L.np - P->n, true);
    const SweepArgs<T> a = make_sweep_args<T>(P, layer, color);
    const bool padded = L.general;
    if (layer <= 3) {
        if (P->mode == CMG_MODE_GAUSS)
            dispatch_small_layer<T, MODE_GAUSS, PREC_EXACT>(P, a, padded);
        else if (P->prec == CMG_PREC_FAST)
            dispatch_small_layer<T, MODE_MEAN, PREC_FAST>(P, a, padded);
        else
            dispatch_small_layer<T, MODE_MEAN, PREC_EXACT>(P, a, padded);
    } else {
        const dim3 grd(wc, hc, P->B);
        // one CTA per patch: 128 threads at level 4 (15 rows, 64 planes), 256 above
        const int nt = layer >= 5 ? 256 : 128;
        if (P->mode == CMG_MODE_GAUSS) {
            if (padded)
                klaunch(P, k_sweep_bpp<T, MODE_GAUSS, SRC_PADDED>, grd, nt, 0, a);
            else
                klaunch(P, k_sweep_bpp<T, MODE_GAUSS, SRC_INPLACE>, grd, nt, 0, a);
        } else {
            if (padded)
                klaunch(P, k_sweep_bpp<T, MODE_MEAN, SRC_PADDED>, grd, nt, 0, a);
            else
                klaunch(P, k_sweep_bpp<T, MODE_MEAN, SRC_INPLACE>, grd, nt, 0, a);
        }
    }
    P->enq += 1;
    stamp(P, 10 * layer + color);
}

template <typename T>
__global__ void k_copy(const T* __restrict__ src, T* __restrict__ dst, long long N, const ImgState* st) {
    pdl_sync();
    const int b = blockIdx.y;
    if (st[b].done) return;
    const long long off = (long long)b * N;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x)
        dst[off + e] = src[off + e];
}

template <typename T>
void enqueue_copy_prev(cmg_plan* P) {
    const int blocks = (int)std::min<long long>((P->N + 255) / 256, 2048);
    klaunch(P, k_copy<T>, dim3(blocks, P->B), 256, 0, (const T*)P->u, (T*)P->uprev, P->N, P->st);
    P->enq += 1;
}

inline int buf_index(const cmg_plan* P, const void* u) {
    for (int i = 0; i < 3; ++i)
        if (u == P->ubuf[i]) return i;
    return 0;
}

inline TraceArgs make_trace_args(const cmg_plan* P, double* eonly, double* raw5) {
    TraceArgs ta;
    ta.energy = P->tr[0];
    ta.rel_e = P->tr[1];
    ta.rel_u = P->tr[2];
    ta.psnr = P->tr[3];
    ta.seconds = P->tr[4];
    ta.cap = P->cap;
    ta.ndone = P->ndone;
    ta.eonly = eonly;
    ta.raw5 = raw5;
    return ta;
}

inline EnergyFin make_energy_fin(const cmg_plan* P, const TraceArgs& ta, int initial, int buf) {
    EnergyFin fz;
    fz.tr = ta;
    fz.P = P->P;
    fz.stw = P->st;
    fz.tickets = P->fused_finalize ? P->tickets : nullptr;
    fz.img_ticket = P->tickets + P->B;
    fz.initial = initial;
    fz.cond = P->cur_cond;
    fz.B = P->B;
    fz.buf = buf;
    return fz;
}

template <typename T>
void enqueue_energy_ptrs(cmg_plan* P, const void* u, const void* uprev, bool has_ref, double* eonly, int initial,
                         double* raw5, long long e_lo, long long e_hi) {
    if (P->egeneral) enqueue_pad<T>(P, u, P->epad, P->eH, P->eW, P->epstride, 1, 1, !initial && !eonly);
    EnergyArgs ea;
    ea.u = u;
    ea.f = P->f;
    ea.uprev = uprev;
    ea.ref = has_ref ? P->ref : nullptr;
    ea.upad = P->epad;
    ea.istride = P->N;
    ea.pstride = P->epstride;
    ea.m = P->m;
    ea.n = P->n;
    ea.W = P->eW;
    ea.mode = P->mode;
    ea.nbx = P->nbx;
    ea.ncb = P->ncb;
    ea.e_lo = e_lo;
    ea.e_hi = e_hi < 0 ? P->N : e_hi;
    ea.partials = P->partials;
    ea.st = P->st;
    const TraceArgs ta = make_trace_args(P, eonly, raw5);
    EnergyFin fz = make_energy_fin(P, ta, initial, buf_index(P, u));
    if (P->egeneral)
        klaunch(P, k_energy<T, SRC_PADDED>, dim3(P->nbx, P->B), 256, 0, ea, fz);
    else if (P->eb_px == 1)
        klaunch(P, k_energy_bulk<T, 1>, dim3(P->nbx, P->B), 288, eb_smem_bytes<T, 1>(P->eb_ns), ea, fz, P->eb_H,
                                                                                                   P->eb_ns);
    else if (P->eb_px == 2)
        klaunch(P, k_energy_bulk<T, 2>, dim3(P->nbx, P->B), 288, eb_smem_bytes<T, 2>(P->eb_ns), ea, fz, P->eb_H,
                                                                                                   P->eb_ns);
    else if (std::is_same<T, float>::value && P->eb_px == 4)
        klaunch(P, k_energy_bulk<float, 4>, dim3(P->nbx, P->B), 288, eb_smem_bytes<float, 4>(P->eb_ns), ea, fz,
                P->eb_H, P->eb_ns);
    else if (P->energy_nt == 512)  // shorter per-thread column walks, still one wave (2 CTAs/SM)
        klaunch(P, k_energy<T, SRC_INPLACE, 512>, dim3(P->nbx, P->B), 512, 0, ea, fz);
    else
        klaunch(P, k_energy<T, SRC_INPLACE>, dim3(P->nbx, P->B), 256, 0, ea, fz);
    stamp(P, 90);
    if (!P->fused_finalize) {
        klaunch(P, k_finalize, P->B, 256, 0, P->partials, P->nbx, P->P, P->st, ta, initial, buf_index(P, u));
        P->enq += 1;
        stamp(P, 91);
    }
    P->enq += 1;
}

template <typename T>
void enqueue_energy(cmg_plan* P, bool has_ref, double* eonly, int initial) {
    enqueue_energy_ptrs<T>(P, P->u, P->uprev, has_ref, eonly, initial, nullptr, 0, -1);
}

template <typename T>
struct L1Tile;
template <>
struct L1Tile<float> {
    static constexpr int TH = 32, TW = 64;
};
template <>
struct L1Tile<double> {
    static constexpr int TH = 32, TW = 32;
};

template <typename T, int MODE, int PREC>
void launch_l1_tile(cmg_plan* P, const FusedArgs<T>& a) {
    if constexpr (std::is_same<T, float>::value && MODE == MODE_MEAN && PREC == PREC_FAST) {
        if (P->l1x2) {  // packed fp32x2 variant
            auto go = [&](auto kern, auto th, auto tw, int nt) {
                constexpr int TH = decltype(th)::value, TW = decltype(tw)::value;
                using G = L1Geom<float, TH, TW>;
                const size_t smem = sizeof(float) * (2 + (P->l1x2 >= 11 ? 4 : 8) * G::PLANE);
                smem_attr(kern, smem);
                const dim3 grd((P->n + TW - 1) / TW, (P->m + TH - 1) / TH, P->B);
                klaunch(P, kern, grd, nt, smem, a);
            };
            using I56 = std::integral_constant<int, 56>;
            using I120 = std::integral_constant<int, 120>;
            using I88 = std::integral_constant<int, 88>;
            // 1: interior fast path (default), 2: Newton rsqrt on the diagonals, 3: generic loop only,
            // 4: 56 x 120 tiles, 5: 88 x 88 tiles (192 threads), 11 / 12: f read from global memory;
            // EF: the energy-fused instantiation (its extra registers stay out of the plain one)
            auto sel = [&](auto ef) {
                constexpr bool EF = decltype(ef)::value;
                switch (P->l1x2) {
                    case 2: go(k_l1_x2<56, 56, 1, true, 256, false, EF>, I56{}, I56{}, 256); break;
                    case 3: go(k_l1_x2<56, 56, 0, false, 256, false, EF>, I56{}, I56{}, 256); break;
                    case 4: go(k_l1_x2<56, 120, 0, true, 256, false, EF>, I56{}, I120{}, 256); break;
                    case 5: go(k_l1_x2<88, 88, 0, true, 192, false, EF>, I88{}, I88{}, 192); break;
                    case 6: go(k_l1_x2<56, 120, 0, false, 256, false, EF>, I56{}, I120{}, 256); break;
                    case 7: go(k_l1_x2<56, 120, 0, true, 512, false, EF>, I56{}, I120{}, 512); break;
                    case 8: go(k_l1_x2<120, 56, 0, true, 256, false, EF>, I120{}, I56{}, 256); break;
                    case 11: go(k_l1_x2<56, 120, 0, true, 256, true, EF>, I56{}, I120{}, 256); break;
                    case 12: go(k_l1_x2<56, 56, 0, true, 256, true, EF>, I56{}, I56{}, 256); break;
                    default: go(k_l1_x2<56, 56, 0, true, 256, false, EF>, I56{}, I56{}, 256); break;
                }
            };
            if (a.efuse)
                sel(std::true_type{});
            else
                sel(std::false_type{});
            return;
        }
    }
    auto go = [&](auto th, auto tw) {
        constexpr int TH = decltype(th)::value, TW = decltype(tw)::value;
        using G = L1Geom<T, TH, TW>;
        const size_t smem = 2 * sizeof(T) * 4 * G::PLANE;
        const dim3 grd((P->n + TW - 1) / TW, (P->m + TH - 1) / TH, P->B);
        if constexpr (std::is_same<T, double>::value && MODE == MODE_MEAN && PREC == PREC_EXACT) {
            // branch-free pixel code (cmg_l1loop.cuh): one inner iteration, sequential plane mean (no
            // single-patch colour class: images of 4+ pixels per side)
            if (P->l1_loop && P->hostP.inner == 1 && P->m >= 4 && P->n >= 4) {
                auto kern = k_l1_tile<T, MODE, PREC, TH, TW, true>;
                smem_attr(kern, smem);
                klaunch(P, kern, grd, 256, smem, a);
                return;
            }
        }
        auto kern = k_l1_tile<T, MODE, PREC, TH, TW>;
        smem_attr(kern, smem);
        klaunch(P, kern, grd, 256, smem, a);
    };
    using IH = std::integral_constant<int, L1Tile<T>::TH>;
    using IW = std::integral_constant<int, L1Tile<T>::TW>;
    if constexpr (std::is_same<T, double>::value) {
        if (P->l1_th == 28) {  // 28 x 64 tiles: 37 x 16 = 592 CTAs = 4 per SM at 1024^2
            go(std::integral_constant<int, 28>{}, std::integral_constant<int, 64>{});
            return;
        }
    }
    if (P->l1_wide)  // 32 x 64 tiles: fewer CTAs (one wave at 1024^2 fp64), less halo per pixel
        go(std::integral_constant<int, 32>{}, std::integral_constant<int, 64>{});
    else
        go(IH{}, IW{});
}

// shared-memory tile configs of the coarse fused levels (patches per tile
// side TP, lanes per patch TS, threads per CTA NT)
template <typename T, int LAYER>
struct CoarseCfg;
template <>
struct CoarseCfg<float, 2> {
    // 24 x 24 patches: 70 KB SMEM, 3 CTAs/SM (16384^2 level 2: 1.31 ms with 32, 1.17 with 24,
    // 1.42 with 16 -- halo recompute (30/24)^2 = 1.56x vs occupancy)
    static constexpr int TP = 24, TS = 1, NT = 256;
};
template <>
struct CoarseCfg<double, 2> {
    static constexpr int TP = 16, TS = 4, NT = 256;
};
template <>
struct CoarseCfg<float, 3> {
    static constexpr int TP = 8, TS = 8, NT = 256;
};
template <>
struct CoarseCfg<double, 3> {
    static constexpr int TP = 4, TS = 8, NT = 128;
};

template <typename T, int LAYER, int MODE, int PREC, bool FS>
void launch_coarse_v(cmg_plan* P, const FusedArgs<T>& a) {
    using C = CoarseCfg<T, LAYER>;
    using G = CoarseGeom<T, LAYER, C::TP>;
    const size_t smem = 128 + (FS ? 1 : 2) * sizeof(T) * G::CELLS_AL + sizeof(PlaneLin) * (G::NPL + 2) + 16;
    auto kern = k_coarse_tile<T, LAYER, MODE, PREC, C::TP, C::TS, C::NT, FS>;
    smem_attr(kern, smem);
    const Level& L = P->lv[LAYER];
    const dim3 grd((L.nj + C::TP - 1) / C::TP, (L.mj + C::TP - 1) / C::TP, P->B);
    int bi = -1;
    for (int i = 0; i < 3; ++i)
        if (a.uin == P->ubuf[i]) bi = i;
    const bool tma = P->tma_ok[LAYER] && bi >= 0;
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof(dummy));
    klaunch(P, kern, grd, C::NT, smem, a, tma ? P->tmap[LAYER][bi] : dummy, tma ? P->tmap[LAYER][3] : dummy,
                                          tma ? 1 : 0);
}

template <typename T, int LAYER, int MODE, int PREC>
void launch_coarse(cmg_plan* P, const FusedArgs<T>& a) {
    using C = CoarseCfg<T, LAYER>;
    if constexpr (C::TS == 1 && MODE == MODE_MEAN && PREC == PREC_FAST) {
        if (a.fsum) {  // per-patch f sums: u only in shared memory
            launch_coarse_v<T, LAYER, MODE, PREC, true>(P, a);
            return;
        }
    }
    launch_coarse_v<T, LAYER, MODE, PREC, false>(P, a);
}

// encoded as box_width * 4096 + box_height
template <typename T>
inline int coarse_region_impl(int layer) {
    using G2 = CoarseGeom<T, 2, CoarseCfg<T, 2>::TP>;
    using G3 = CoarseGeom<T, 3, CoarseCfg<T, 3>::TP>;
    return layer == 2 ? G2::BW * 4096 + G2::RD : G3::BW * 4096 + G3::RD;
}

// levels 2-3: two launches (patch-row parity 0, then 1), each running its two
// colours in a shared-memory window (cmg_rowpair.cuh); X -> Y
template <typename T, int LAYER, int MODE, int PREC, int TS, int NT = 256>
void launch_rowpair(cmg_plan* P, const T* X, T* Y) {
    using G = RowPairGeom<LAYER, TS, NT>;
    const Level& L = P->lv[LAYER];
    RowPairArgs<T> r;
    r.X = X;
    r.Y = Y;
    r.nj = L.nj;
    r.ntiles = (L.nj + G::TPC - 1) / G::TPC;
    // u window + f of the patch row (no f rows with per-patch f sums)
    const bool fs = P->fsum[LAYER] != nullptr && MODE == MODE_MEAN && PREC == PREC_FAST;
    const size_t smem = sizeof(T) * (G::ROWS + (fs ? 0 : G::S)) * G::WIN;
    auto kern = k_rowpair<T, LAYER, MODE, PREC, TS, NT>;
    smem_attr(kern, smem);
    for (int p = 0; p < 2; ++p) {
        const int rows = (L.mj - p + 1) / 2;
        if (rows <= 0) continue;
        r.c0 = make_sweep_args<T>(P, LAYER, 2 * p);
        r.c1 = make_sweep_args<T>(P, LAYER, 2 * p + 1);
        klaunch(P, kern, dim3(r.ntiles, rows, P->B), G::NT, smem, r);
        if (p == 0) {
            stamp(P, 10 * LAYER + 8);
        } else {
            P->enq += 1;  // the caller counts one launch per level
        }
    }
}

// the same launches with bulk-copy staging and bulk-store write-back
// (k_rowpair_tma; n*sizeof(T) % 16 == 0)
template <typename T, int LAYER, int MODE, int PREC, int TS, int NT = 256>
void launch_rowpair_tma(cmg_plan* P, const T* X, T* Y) {
    using G = RowPairGeom<LAYER, TS, NT, 16 / (int)sizeof(T)>;
    const Level& L = P->lv[LAYER];
    RowPairArgs<T> r;
    r.X = X;
    r.Y = Y;
    r.nj = L.nj;
    r.ntiles = (L.nj + G::TPC - 1) / G::TPC;
    const bool fs = P->fsum[LAYER] != nullptr && MODE == MODE_MEAN && PREC == PREC_FAST;
    const size_t smem = sizeof(T) * (G::ROWS + (fs ? 0 : G::S)) * G::WIN;
    auto kern = k_rowpair_tma<T, LAYER, MODE, PREC, TS, NT>;
    smem_attr(kern, smem);
    for (int p = 0; p < 2; ++p) {
        const int rows = (L.mj - p + 1) / 2;
        if (rows <= 0) continue;
        r.c0 = make_sweep_args<T>(P, LAYER, 2 * p);
        r.c1 = make_sweep_args<T>(P, LAYER, 2 * p + 1);
        klaunch(P, kern, dim3(r.ntiles, rows, P->B), G::NT, smem, r);
        if (p == 0) {
            stamp(P, 10 * LAYER + 8);
        } else {
            P->enq += 1;  // the caller counts one launch per level
        }
    }
}

// persistent bulk-copy variant (one thread per patch, fast mean + f sums)
template <typename T, int LAYER, int NT, int STAGES, int TPC_ = 0>
void launch_rowpair_bulk_s(cmg_plan* P, const T* X, T* Y) {
    using G = RowPairGeom<LAYER, 1, NT, 16 / (int)sizeof(T), TPC_>;
    const Level& L = P->lv[LAYER];
    RowPairArgs<T> r;
    r.X = X;
    r.Y = Y;
    r.nj = L.nj;
    r.ntiles = (L.nj + G::TPC - 1) / G::TPC;
    const size_t smem = STAGES * sizeof(T) * G::ROWS * G::WIN;
    auto kern = k_rowpair_bulk<T, LAYER, NT, STAGES, TPC_>;
    smem_attr(kern, smem);
    int occ = 1, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P->device);
    for (int p = 0; p < 2; ++p) {
        const int rows = (L.mj - p + 1) / 2;
        if (rows <= 0) continue;
        r.c0 = make_sweep_args<T>(P, LAYER, 2 * p);
        r.c1 = make_sweep_args<T>(P, LAYER, 2 * p + 1);
        const long long items = (long long)rows * r.ntiles * P->B;
        const int grid = (int)std::min<long long>(items, (long long)nsm * std::max(1, occ));
        klaunch(P, kern, dim3(grid), NT, smem, r, rows, P->B);
        if (p == 0) {
            stamp(P, 10 * LAYER + 8);
        } else {
            P->enq += 1;  // the caller counts one launch per level
        }
    }
}

template <typename T, int LAYER, int NT, int TPC_ = 0>
void launch_rowpair_bulk(cmg_plan* P, const T* X, T* Y) {
    if (P->rp_stages == 1)
        launch_rowpair_bulk_s<T, LAYER, NT, 1, TPC_>(P, X, Y);
    else
        launch_rowpair_bulk_s<T, LAYER, NT, 2, TPC_>(P, X, Y);
}

template <typename T, int MODE, int PREC>
void dispatch_rowpair(cmg_plan* P, int layer, const FusedArgs<T>& a) {
    // one thread per patch (fast mean with per-patch f sums; large jobs): a
    // ~64 KB window of one patch row per CTA
    if constexpr (MODE == MODE_MEAN && PREC == PREC_FAST) {
        if (((P->rp1 >> (layer - 2)) & 1) && a.fsum) {
            constexpr int NT1 = 64;
            if (P->rp_bulk && ((size_t)P->n * sizeof(T)) % 16 == 0) {
                // narrow images (64 x 512^2): one 172-patch tile per level-2 patch row with
                // 128 threads instead of three 62-patch tiles with 32 (87 -> 78 us per visit;
                // the same at level 3, one 74-patch tile with 64 threads: 116 vs 111 us for
                // the per-colour team kernels, not kept)
                if (sizeof(T) == 4 && P->rp_nt2 == 172 && layer == 2 && P->lv[2].nj <= 172) {
                    launch_rowpair_bulk<T, 2, 128, 172>(P, a.uin, a.uout);
                    return;
                }
                if (sizeof(T) == 4 && P->rp_nt == 128) {
                    if (layer == 2)
                        launch_rowpair_bulk<T, 2, 128>(P, a.uin, a.uout);
                    else
                        launch_rowpair_bulk<T, 3, 128>(P, a.uin, a.uout);
                } else if (P->rp_nt == 32) {
                    if (layer == 2)
                        launch_rowpair_bulk<T, 2, 32>(P, a.uin, a.uout);
                    else
                        launch_rowpair_bulk<T, 3, 32>(P, a.uin, a.uout);
                } else if (layer == 2) {
                    launch_rowpair_bulk<T, 2, NT1>(P, a.uin, a.uout);
                } else {
                    launch_rowpair_bulk<T, 3, NT1>(P, a.uin, a.uout);
                }
                return;
            }
            if (layer == 2)
                launch_rowpair<T, 2, MODE, PREC, 1, NT1>(P, a.uin, a.uout);
            else
                launch_rowpair<T, 3, MODE, PREC, 1, NT1>(P, a.uin, a.uout);
            return;
        }
    }
    // team sizes: level 2 {4, 8} lanes per patch (P->rp_ts2), level 3 {8, 16}
    if (P->rp_tma && ((size_t)P->n * sizeof(T)) % 16 == 0) {
        // level 2 with 128-thread CTAs: twice the CTAs, evener SM load (1024^2 fp64 exact:
        // 27.2 -> 25.5 us per visit; 64 threads: 29.0 us; level 3 with 128 threads: 25.5 -> 26.6 us)
        if (layer == 2 && P->rp_ts2 < 8 && P->rp_tnt == 128) {
            launch_rowpair_tma<T, 2, MODE, PREC, 4, 128>(P, a.uin, a.uout);
            return;
        }
        if (layer == 2) {
            if (P->rp_ts2 >= 8)
                launch_rowpair_tma<T, 2, MODE, PREC, 8>(P, a.uin, a.uout);
            else
                launch_rowpair_tma<T, 2, MODE, PREC, 4>(P, a.uin, a.uout);
        } else {
            if (P->ts3 >= 16)
                launch_rowpair_tma<T, 3, MODE, PREC, 16>(P, a.uin, a.uout);
            else
                launch_rowpair_tma<T, 3, MODE, PREC, 8>(P, a.uin, a.uout);
        }
        return;
    }
    if (layer == 2) {
        if (P->rp_ts2 >= 8)
            launch_rowpair<T, 2, MODE, PREC, 8>(P, a.uin, a.uout);
        else
            launch_rowpair<T, 2, MODE, PREC, 4>(P, a.uin, a.uout);
    } else {
        if (P->ts3 >= 16)
            launch_rowpair<T, 3, MODE, PREC, 16>(P, a.uin, a.uout);
        else
            launch_rowpair<T, 3, MODE, PREC, 8>(P, a.uin, a.uout);
    }
}

template <typename T, int MODE, int PREC>
void dispatch_fused(cmg_plan* P, int layer, const FusedArgs<T>& a) {
    if (layer >= 2 && ((P->rowpair >> (layer - 2)) & 1)) {
        dispatch_rowpair<T, MODE, PREC>(P, layer, a);
        return;
    }
    if (layer == 1)
        launch_l1_tile<T, MODE, PREC>(P, a);
    else if (layer == 2)
        launch_coarse<T, 2, MODE, PREC>(P, a);
    else
        launch_coarse<T, 3, MODE, PREC>(P, a);
}


// one fused level visit uin -> uout; efuse_prev != nullptr: energy-fused
// level-1 visit whose input is the cycle input u_g and efuse_prev is u_{g-1}
template <typename T>
void enqueue_fused_level_x(cmg_plan* P, int layer, const void* uin, void* uout, const void* efuse_prev,
                           bool has_ref) {
    const Level& L = P->lv[layer];
    FusedArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.uin = (const T*)uin;
    a.uout = (T*)uout;
    a.efuse = efuse_prev != nullptr;
    if (a.efuse) {
        a.uprev = (const T*)efuse_prev;
        a.ref = has_ref ? (const T*)P->ref : nullptr;
        a.partials = P->partials;
        a.mode = P->mode;
        a.fz = make_energy_fin(P, make_trace_args(P, nullptr, nullptr), 2, buf_index(P, uin));
    }
    a.f = (const T*)P->f;
    a.istride = P->N;
    a.m = P->m;
    a.n = P->n;
    a.mj = L.mj;
    a.nj = L.nj;
    a.tiles_c = 0;  // set per variant by launch_fused
    a.dbg = P->dbg;
    a.nz = -0.0f;
    for (int c = 0; c < 4; ++c) {
        const int p = c >> 1, q = c & 1;
        a.hc[c] = (L.mj - p + 1) / 2;
        a.wc[c] = (L.nj - q + 1) / 2;
    }
    a.P = P->P;
    a.st = P->st;
    a.fsum = (layer >= 2 && layer <= 3) ? P->fsum[layer] : nullptr;
    a.fs_img = (long long)L.mj * L.nj;
    a.fs_ld = L.nj;
    if (P->mode == CMG_MODE_GAUSS)
        dispatch_fused<T, MODE_GAUSS, PREC_EXACT>(P, layer, a);
    else if (P->prec == CMG_PREC_FAST)
        dispatch_fused<T, MODE_MEAN, PREC_FAST>(P, layer, a);
    else
        dispatch_fused<T, MODE_MEAN, PREC_EXACT>(P, layer, a);
    P->enq += 1;
    stamp(P, 100 + layer);
}

template <typename T>
void enqueue_fused_level(cmg_plan* P, int layer, const void* uin, void* uout) {
    enqueue_fused_level_x<T>(P, layer, uin, uout, nullptr, false);
}

// Two V-cycles per graph body with a 3-buffer rotation: fused levels write
// into a buffer that is neither their input nor the cycle's u_prev, so rel_u
// needs no copy, and after the two cycles u is back in ubuf[0].
template <typename T>
void enqueue_body_fused(cmg_plan* P, int full, bool has_ref) {
    std::vector<int> seq;
    for (int j = 1; j <= P->layers; ++j) seq.push_back(j);
    if (full)
        for (int j = P->layers - 1; j >= 1; --j) seq.push_back(j);
    auto fusedj = [&](int j) { return j <= 3 && ((P->fuse_mask >> (j - 1)) & 1); };
    int nf = 0;
    for (int j : seq) nf += fusedj(j);
    int cur = 0;
    for (int half = 0; half < 2; ++half) {
        const int prev = cur;
        const int target = (half == 0) ? 1 : 0;
        int other = 3 - prev - target;
        bool first = true;
        for (int j : seq) {
            if (fusedj(j)) {
                int out;
                if (first) {
                    out = (nf & 1) ? target : other;
                    first = false;
                } else {
                    out = 3 - prev - cur;
                }
                enqueue_fused_level<T>(P, j, P->ubuf[cur], P->ubuf[out]);
                cur = out;
            } else {
                void* save = P->u;
                P->u = P->ubuf[cur];
                for (int c = 0; c < 4; ++c) enqueue_sweep<T>(P, j, c);
                P->u = save;
            }
        }
        enqueue_energy_ptrs<T>(P, P->ubuf[cur], P->ubuf[prev], has_ref, nullptr, 0, nullptr, 0, -1);
    }
}

// Energy-fused cycles.  The level-1 kernel of cycle g+1 also computes and
// finalizes the energy of its input u_g (trace, stopping rule, WHILE
// condition), so a cycle has no separate energy pass.  Buffer roles per cycle:
// X = input u_g, Pv = u_{g-1} (read by that level-1 kernel for rel_u), Z = the
// third buffer.  Level 1: X -> Z; the later fused levels alternate Z <-> Pv
// (X stays intact: a stopped image's later levels copy u_g from it); in-place
// levels run on the current buffer.  The next cycle's (X, Pv) = (output, X).
// A graph body holds the 2 or 3 cycles after which the roles return to
// (0, 1, 2).  Stopping: once cycle g is finalized as the last one, that image's
// later levels copy u_g along, so after the body it is in buffer 0.
template <typename T>
void enqueue_body_efused(cmg_plan* P, int full, bool has_ref) {
    std::vector<int> seq;
    for (int j = 1; j <= P->layers; ++j) seq.push_back(j);
    if (full)
        for (int j = P->layers - 1; j >= 1; --j) seq.push_back(j);
    auto fusedj = [&](int j) { return j <= 3 && ((P->fuse_mask >> (j - 1)) & 1); };
    const int per = efused_cycles_per_body(P, full);
    int X = 0, Pv = 1, Z = 2;
    for (int h = 0; h < per; ++h) {
        int cur = X;
        bool first = true;
        for (int j : seq) {
            if (fusedj(j)) {
                const int out = first ? Z : ((cur == Z) ? Pv : Z);
                enqueue_fused_level_x<T>(P, j, P->ubuf[cur], P->ubuf[out], first ? P->ubuf[Pv] : nullptr, has_ref);
                first = false;
                cur = out;
            } else {
                void* save = P->u;
                P->u = P->ubuf[cur];
                for (int c = 0; c < 4; ++c) enqueue_sweep<T>(P, j, c);
                P->u = save;
            }
        }
        Pv = X;
        X = cur;
        Z = 3 - X - Pv;
    }
}

template <typename T>
void enqueue_collect(cmg_plan* P) {
    const int blocks = (int)std::min<long long>((P->N + 255) / 256, 1024);
    klaunch(P, k_collect<T>, dim3(blocks, P->B), 256, 0, (T*)P->ubuf[0], (const T*)P->ubuf[1], (const T*)P->ubuf[2],
            P->N, (const ImgState*)P->st);
    P->enq += 1;
}

template <typename T>
void enqueue_fpads(cmg_plan* P) {
    for (int j = 1; j <= P->layers; ++j) {
        Level& L = P->lv[j];
        if (L.general) enqueue_pad<T>(P, P->f, L.fpad, L.H, L.W, L.pstride, 1 + L.mp - P->m, 1 + L.np - P->n, false);
    }
}

// k_energy_bulk geometry: band height H (halved until the items fill the
// resident CTAs); returns CTAs per image
template <typename T, int PX>
int energy_bulk_occ(int ns) {
    const size_t sm = eb_smem_bytes<T, PX>(ns);
    cudaFuncSetAttribute(k_energy_bulk<T, PX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int bps = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_energy_bulk<T, PX>, 288, sm);
    return std::max(1, bps);
}
template <typename T>
int energy_bulk_cfg_impl(int batch, int m, int n, int px, int ns, int* H_out) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int bps = 1;
    if (px == 1) bps = energy_bulk_occ<T, 1>(ns);
    if (px == 2) bps = energy_bulk_occ<T, 2>(ns);
    if (px == 4) bps = energy_bulk_occ<float, 4>(ns);
    const long long per_img = std::max(1LL, (long long)nsm * bps / batch);
    const long long ncb = (n + 256 * px - 1) / (256 * px);
    int H = 32;
    while (H > 2 && ((m + H - 1) / H) * ncb < per_img) H /= 2;
    *H_out = H;
    return (int)std::max(1LL, std::min(per_img, ((m + H - 1) / H) * ncb));
}

}  // namespace cmg

#define CMG_INSTANTIATE(T)                                                          \
    template void cmg::enqueue_sweep<T>(cmg_plan*, int, int);                       \
    template void cmg::enqueue_energy<T>(cmg_plan*, bool, double*, int);            \
    template void cmg::enqueue_copy_prev<T>(cmg_plan*);                             \
    template void cmg::enqueue_fpads<T>(cmg_plan*);                             \
    template void cmg::enqueue_fsums<T>(cmg_plan*);                             \
    template void cmg::enqueue_fused_level<T>(cmg_plan*, int, const void*, void*);  \
    template void cmg::enqueue_energy_ptrs<T>(cmg_plan*, const void*, const void*, bool, double*, int, double*, \
                                              long long, long long);                                   \
    template void cmg::enqueue_body_fused<T>(cmg_plan*, int, bool);                  \
    template void cmg::enqueue_body_efused<T>(cmg_plan*, int, bool);                 \
    template void cmg::enqueue_collect<T>(cmg_plan*);                                \
    template <>                                                                     \
    int cmg::coarse_region<T>(int layer) {                                          \
        return cmg::coarse_region_impl<T>(layer);                                   \
    }                                                                               \
    template <>                                                                     \
    int cmg::energy_bulk_cfg<T>(int batch, int m, int n, int px, int ns, int* H) {  \
        return cmg::energy_bulk_cfg_impl<T>(batch, m, n, px, ns, H);                \
    }
