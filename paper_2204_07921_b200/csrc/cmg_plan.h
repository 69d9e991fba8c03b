// cmg_plan.h -- the solver plan (device buffers, graph, statistics) shared by
// the host runtime (cmg.cu) and the per-dtype launch units (cmg_f64/f32.cu).
#pragma once

#include <cuda.h>
#include <cstring>
#include <utility>
#include <cuda_runtime.h>
#include <mutex>
#include <vector>
#include <set>
#include <utility>

#include "../../include/cmg.h"
#include "cmg_kernels.cuh"

namespace cmg {

// One level of the hierarchy (hierarchy.Partition, hierarchy.py:29-73).
struct Level {
    int layer = 0, s = 0, r = 0, mj = 0, nj = 0, mp = 0, np = 0;
    bool general = false;  // needs numpy's iterated/singleton reflection -> padded snapshot
    int H = 0, W = 0;
    long long pstride = 0;
    void* fpad = nullptr;
};

}  // namespace cmg

struct cmg_plan {
    int m = 0, n = 0, B = 0, layers = 0, mode = 0, dtype = 0, prec = 0, device = 0;
    size_t esz = 8;
    long long N = 0;
    cudaStream_t stream = nullptr;
    void *u = nullptr, *uprev = nullptr, *f = nullptr, *ref = nullptr, *upad = nullptr, *epad = nullptr;
    size_t upad_elems = 0;
    bool egeneral = false;
    int eH = 0, eW = 0;
    long long epstride = 0;
    cmg::Level lv[7];
    double* partials = nullptr;
    int nbx = 1;
    int ncb = 1;  // k_energy column chunks (nbx = row bands * ncb)
    int eb_px = 0, eb_ns = 4, eb_H = 32;  // k_energy_bulk<T, eb_px> (0: off)
    cmg::ImgState* st = nullptr;
    int* ndone = nullptr;
    int* iters = nullptr;
    double* eonly = nullptr;
    double* raw5 = nullptr;  // [B][5] strip-mode partial sums
    cmg::SolveParams* P = nullptr;
    cmg::SolveParams hostP;  // host copy of the current parameters (kernel-argument constants)
    double galpha = -1.0;     // parameters baked into the cached graph
    int ginner = -1;
    double* tr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int cap = 0;
    // kernel variants
    int ts2 = 4, ts3 = 16;
    int dbg = 0;
    bool fused_finalize = true;       // energy kernel's last CTA runs the finalize (+ WHILE condition)
    int* tickets = nullptr;           // [B] + 1 counters of that scheme
    unsigned long long cur_cond = 0;  // conditional handle while capturing the WHILE body
    unsigned long long* stamps = nullptr;  // CMG_STAMPS diagnostics buffer
    int stamps_cap = 0;
    int l1x2 = 1;  // packed fp32x2 level-1 kernel (fp32 fast mean); variants in launch_l1_tile
    bool tma_ok[4] = {false, false, false, false};
    CUtensorMap tmap[4][4];  // [level][buffer 0..2 = u rotation, 3 = f]
    // graphs
    cudaGraphExec_t exec = nullptr;
    int gkey = -1;
    bool use_while = true;
    int nodes_per_cycle = 0;
    bool no_graph = false;  // CMG_NO_GRAPH=1: no graph at all (kernels visible to ncu)
    // stats
    long long launches = 0;
    int cycles_run = 0;
    float dev_ms = 0.f;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int enq = 0;  // kernels enqueued since last reset
    // fused-level path (all four colours of a level in one tile kernel)
    bool fused = false;
    int fuse_mask = 7;  // bit j-1: level j runs as one fused tile kernel (bit 0 required)
    void* ubuf[3] = {nullptr, nullptr, nullptr};  // rotation buffers (ubuf[0]=u, ubuf[1]=uprev)
    int pcap = 0;           // partials capacity (images x energy CTAs)
    bool efuse = false;     // energy-fused cycles (enqueue_body_efused; CMG_EFUSE=0: off)
    cudaError_t launch_err = cudaSuccess;  // first failed checked launch
    int rowpair = 3;        // bit j-2: level j (2, 3) runs as two row-parity launches (k_rowpair)
    bool l1_wide = false;   // k_l1_tile with 32 x 64 tiles (CMG_L1_WIDE)
    int rp_tnt = 128;       // threads per CTA of the bulk-staged level-2 team row-parity kernel (CMG_RP_TNT=256)
    int rp_nt2 = 0;         // level-2 bulk row-parity kernel: 172 = one 172-patch tile per row (CMG_RP_NT2)
    int l1_th = 0;          // fp64 level-1 tile height override (CMG_L1_TH=28: 28 x 64 tiles)
    bool l1_loop = true;    // fp64 exact mean level 1: branch-free sqrt/div pixel code of cmg_l1loop.cuh
                            // (CMG_L1_LOOP=0: library sqrt/div)
    int rp_ts2 = 4;         // lanes per patch of the level-2 row-parity kernel (CMG_RP_TS2)
    int rp1 = 0;            // bit j-2: level j's row-parity kernel runs one thread per patch (CMG_RP1)
    int rp_tma = 1;         // k_rowpair with bulk-copy staging / bulk-store write-back (CMG_RP_TMA)
    int rp_bulk = 1;        // ... as the persistent bulk-copy kernel (CMG_RP_BULK)
    int rp_stages = 1;      // shared-memory stages of that kernel (CMG_RP_STAGES: 1 or 2; 1 = more CTAs per SM, faster)
    int rp_nt = 64;         // threads per CTA of that kernel (CMG_RP_NT: 32, 64 or 128 [fp32])
    int energy_nt = 512;    // k_energy CTA size (CMG_ENERGY_NT; 512 at <= 64 registers: 1024^2 fp32 3.11 -> 3.04 ms)
    double* fsum[4] = {nullptr, nullptr, nullptr, nullptr};  // [level] per-patch f sums (fast mean, levels 2-3)
    bool use_fsum = true;   // CMG_FSUM=0: f* from f pixels as in exact mode
    bool pdl = true;        // programmatic dependent launch between the cycle's kernels (CMG_PDL=0: off)
};

namespace cmg {
// Launch on the plan's stream; with P->pdl the launch carries programmatic
// stream serialization, so the kernel may be scheduled while its predecessor
// drains (every kernel begins with pdl_sync(), which waits for it).
template <typename... KP, typename... Args>
inline void klaunch(const cmg_plan* P, void (*kern)(KP...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = P->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = P->pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// opt a kernel into its dynamic shared memory on the CURRENT device, once per
// (kernel, device): function attributes are per device, so a process with
// plans on several GPUs needs them set on each
inline void smem_attr_raw(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done.insert({kern, dev}).second)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}
template <typename... KP>
inline void smem_attr(void (*kern)(KP...), size_t smem) {
    smem_attr_raw((const void*)kern, smem);
}

// diagnostics: a 1-thread kernel that appends %globaltimer to a device buffer
// (CMG_STAMPS=1); placed after every node of the cycle to attribute time
static __global__ void k_stamp(unsigned long long* buf, int cap, int tag) {
    pdl_sync();
    const int i = atomicAdd(reinterpret_cast<int*>(buf), 1);
    if (i + 1 < cap) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        buf[1 + i] = (t << 8) | (unsigned)tag;
    }
}

inline void stamp(cmg_plan* P, int tag) {
    if (P->stamps) k_stamp<<<1, 1, 0, P->stream>>>(P->stamps, P->stamps_cap, tag);
}

template <typename T>
void enqueue_sweep(cmg_plan* P, int layer, int color);
template <typename T>
void enqueue_energy(cmg_plan* P, bool has_ref, double* eonly, int initial);
template <typename T>
void enqueue_copy_prev(cmg_plan* P);
template <typename T>
void enqueue_fpads(cmg_plan* P);
template <typename T>
void enqueue_fsums(cmg_plan* P);
template <typename T>
void enqueue_fused_level(cmg_plan* P, int layer, const void* uin, void* uout);
template <typename T>
void enqueue_energy_ptrs(cmg_plan* P, const void* u, const void* uprev, bool has_ref, double* eonly, int initial,
                         double* raw5, long long e_lo, long long e_hi);
template <typename T>
void enqueue_body_fused(cmg_plan* P, int full, bool has_ref);
template <typename T>
void enqueue_body_efused(cmg_plan* P, int full, bool has_ref);
template <typename T>
void enqueue_collect(cmg_plan* P);
inline int efused_out(const cmg_plan* P, int full, int X, int Pv, int Z) {
    int cur = X;
    bool first = true;
    std::vector<int> seq;
    for (int j = 1; j <= P->layers; ++j) seq.push_back(j);
    if (full)
        for (int j = P->layers - 1; j >= 1; --j) seq.push_back(j);
    for (int j : seq) {
        if (!(j <= 3 && ((P->fuse_mask >> (j - 1)) & 1))) continue;
        if (first) {
            cur = Z;
            first = false;
        } else {
            cur = (cur == Z) ? Pv : Z;
        }
    }
    return cur;
}

inline int efused_cycles_per_body(const cmg_plan* P, int full) {
    int X = 0, Pv = 1, Z = 2, k = 0;
    do {
        const int o = efused_out(P, full, X, Pv, Z);
        Pv = X;
        X = o;
        Z = 3 - X - Pv;
        ++k;
    } while (!(X == 0 && Pv == 1) && k < 6);
    return k;
}


template <typename T>
int coarse_region(int layer);
template <typename T>
int energy_bulk_cfg(int batch, int m, int n, int px, int ns, int* H);
template <typename T>
bool make_tmap(CUtensorMap* out, const void* base, int esz, int m, int n, int B, int box);
}  // namespace cmg
