// cmg.cu -- host runtime + C ABI of the B200 multigrid curvature solver.
//
// A plan owns the device images (u, u_prev, f, ref), the per-image solver
// state, the trace buffers and a CUDA graph of the whole outer loop:
//
//     [ WHILE (some image still running) {
//           copy u -> u_prev
//           for j in layer_sequence:           (driver.py:254-258)
//               for colour in COLOR_ORDER:     (driver.py:35, :242)
//                   sweep kernel (in place)
//           energy partials; finalize (trace + stopping rule on device)
//       } ]
//
// The stopping rule is evaluated on the device and fed back into the graph
// through a conditional WHILE node, so one cudaGraphLaunch runs the whole
// denoise (driver.py:296-310) without host round-trips.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cmg.h"
#include "cmg_kernels.cuh"

using namespace cmg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) return fail(CMG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct Level {
    int layer = 0, s = 0, r = 0, mj = 0, nj = 0, mp = 0, np = 0;
    bool general = false;  // needs numpy's iterated/singleton reflection -> padded snapshot
    int H = 0, W = 0;
    long long pstride = 0;
    void* fpad = nullptr;
};

inline bool single_chunk(int len, int pad_after) { return len >= 2 && pad_after <= len - 1; }

}  // namespace

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
    Level lv[7];
    double* partials = nullptr;
    int nbx = 1;
    ImgState* st = nullptr;
    int* ndone = nullptr;
    int* iters = nullptr;
    double* eonly = nullptr;
    SolveParams* P = nullptr;
    double* tr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int cap = 0;
    // graphs
    cudaGraphExec_t exec = nullptr;
    int gkey = -1;
    bool use_while = true;
    int nodes_per_cycle = 0;
    // stats
    long long launches = 0;
    int cycles_run = 0;
    float dev_ms = 0.f;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // launch counter during enqueue
    int enq = 0;
};

namespace {

// ---------------------------------------------------------------------------
// enqueue helpers (used directly and under stream capture)
// ---------------------------------------------------------------------------
template <typename T>
void enqueue_pad(cmg_plan* P, const void* src, void* dst, int H, int W, long long pstride, int bot, int rgt,
                 bool gate) {
    const ImgState* st = gate ? P->st : nullptr;
    int blocks = (int)std::min<long long>((P->N + 255) / 256, 4096);
    k_pad_copy<T><<<dim3(blocks, P->B), 256, 0, P->stream>>>((const T*)src, P->N, (T*)dst, pstride, P->m, P->n, W,
                                                             st);
    k_pad_axis<T><<<dim3((P->n + 127) / 128, P->B), 128, 0, P->stream>>>((T*)dst, pstride, 0, P->m, P->n, H, W,
                                                                         bot, rgt, st);
    k_pad_axis<T><<<dim3((H + 127) / 128, P->B), 128, 0, P->stream>>>((T*)dst, pstride, 1, P->m, P->n, H, W, bot,
                                                                      rgt, st);
    P->enq += 3;
}

template <typename T, int LAYER, int MODE, int PREC>
void launch_tpp(const SweepArgs<T>& a, bool padded, int B, cudaStream_t s) {
    dim3 blk(32, 8);
    dim3 grd((a.wc + 31) / 32, (a.hc + 7) / 8, B);
    if (padded)
        k_sweep_tpp<T, LAYER, MODE, PREC, SRC_PADDED><<<grd, blk, 0, s>>>(a);
    else
        k_sweep_tpp<T, LAYER, MODE, PREC, SRC_INPLACE><<<grd, blk, 0, s>>>(a);
}

template <typename T, int MODE, int PREC>
void dispatch_tpp_layer(const SweepArgs<T>& a, bool padded, int B, cudaStream_t s) {
    switch (a.layer) {
        case 1: launch_tpp<T, 1, MODE, PREC>(a, padded, B, s); break;
        case 2: launch_tpp<T, 2, MODE, PREC>(a, padded, B, s); break;
        default: launch_tpp<T, 3, MODE, PREC>(a, padded, B, s); break;
    }
}

template <typename T>
void enqueue_sweep(cmg_plan* P, int layer, int color) {
    Level& L = P->lv[layer];
    const int p = color >> 1, q = color & 1;
    const int hc = (L.mj - p + 1) / 2, wc = (L.nj - q + 1) / 2;
    if (hc <= 0 || wc <= 0) return;
    if (L.general) enqueue_pad<T>(P, P->u, P->upad, L.H, L.W, L.pstride, 1 + L.mp - P->m, 1 + L.np - P->n, true);
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
    a.flat = (wc == 1);
    a.single = (hc * wc == 1);
    a.P = P->P;
    a.st = P->st;
    const bool padded = L.general;
    if (layer <= 3) {
        if (P->mode == CMG_MODE_GAUSS)
            dispatch_tpp_layer<T, MODE_GAUSS, PREC_EXACT>(a, padded, P->B, P->stream);
        else if (P->prec == CMG_PREC_FAST)
            dispatch_tpp_layer<T, MODE_MEAN, PREC_FAST>(a, padded, P->B, P->stream);
        else
            dispatch_tpp_layer<T, MODE_MEAN, PREC_EXACT>(a, padded, P->B, P->stream);
    } else {
        dim3 grd(wc, hc, P->B);
        if (P->mode == CMG_MODE_GAUSS) {
            if (padded)
                k_sweep_bpp<T, MODE_GAUSS, SRC_PADDED><<<grd, 128, 0, P->stream>>>(a);
            else
                k_sweep_bpp<T, MODE_GAUSS, SRC_INPLACE><<<grd, 128, 0, P->stream>>>(a);
        } else {
            if (padded)
                k_sweep_bpp<T, MODE_MEAN, SRC_PADDED><<<grd, 128, 0, P->stream>>>(a);
            else
                k_sweep_bpp<T, MODE_MEAN, SRC_INPLACE><<<grd, 128, 0, P->stream>>>(a);
        }
    }
    P->enq += 1;
}

template <typename T>
__global__ void k_copy(const T* __restrict__ src, T* __restrict__ dst, long long N, const ImgState* st) {
    const int b = blockIdx.y;
    if (st[b].done) return;
    const long long off = (long long)b * N;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x)
        dst[off + e] = src[off + e];
}

__global__ void k_cond(cudaGraphConditionalHandle h, const int* ndone, int B, int* iters) {
    *iters += 1;
    cudaGraphSetConditional(h, (*ndone < B) ? 1u : 0u);
}

template <typename T>
void enqueue_energy(cmg_plan* P, bool has_ref, double* eonly, int initial) {
    if (P->egeneral) enqueue_pad<T>(P, P->u, P->epad, P->eH, P->eW, P->epstride, 1, 1, !initial && !eonly);
    EnergyArgs ea;
    ea.u = P->u;
    ea.f = P->f;
    ea.uprev = P->uprev;
    ea.ref = has_ref ? P->ref : nullptr;
    ea.upad = P->epad;
    ea.istride = P->N;
    ea.pstride = P->epstride;
    ea.m = P->m;
    ea.n = P->n;
    ea.W = P->eW;
    ea.mode = P->mode;
    ea.nbx = P->nbx;
    ea.partials = P->partials;
    ea.st = P->st;
    if (P->egeneral)
        k_energy<T, SRC_PADDED><<<dim3(P->nbx, P->B), 256, 0, P->stream>>>(ea);
    else
        k_energy<T, SRC_INPLACE><<<dim3(P->nbx, P->B), 256, 0, P->stream>>>(ea);
    TraceArgs ta;
    ta.energy = P->tr[0];
    ta.rel_e = P->tr[1];
    ta.rel_u = P->tr[2];
    ta.psnr = P->tr[3];
    ta.seconds = P->tr[4];
    ta.cap = P->cap;
    ta.ndone = P->ndone;
    ta.eonly = eonly;
    k_finalize<<<P->B, 256, 0, P->stream>>>(P->partials, P->nbx, P->P, P->st, ta, initial);
    P->enq += 2;
}

std::vector<int> layer_sequence(int layers, int full) {
    std::vector<int> s;
    for (int j = 1; j <= layers; ++j) s.push_back(j);
    if (full)
        for (int j = layers - 1; j >= 1; --j) s.push_back(j);
    return s;
}

template <typename T>
void enqueue_cycle_T(cmg_plan* P, int full, bool has_ref) {
    const long long N = P->N;
    int blocks = (int)std::min<long long>((N + 255) / 256, 2048);
    k_copy<T><<<dim3(blocks, P->B), 256, 0, P->stream>>>((const T*)P->u, (T*)P->uprev, N, P->st);
    P->enq += 1;
    for (int j : layer_sequence(P->layers, full))
        for (int c = 0; c < 4; ++c) enqueue_sweep<T>(P, j, c);
    enqueue_energy<T>(P, has_ref, nullptr, 0);
}

void enqueue_cycle(cmg_plan* P, int full, bool has_ref) {
    if (P->dtype == CMG_F64)
        enqueue_cycle_T<double>(P, full, has_ref);
    else
        enqueue_cycle_T<float>(P, full, has_ref);
}

int build_graph(cmg_plan* P, int full, bool has_ref) {
    const int key = full * 2 + (has_ref ? 1 : 0);
    if (P->exec && P->gkey == key) return CMG_OK;
    if (P->exec) {
        cudaGraphExecDestroy(P->exec);
        P->exec = nullptr;
    }
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    if (P->use_while) {
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        alignas(cudaGraphNodeParams) unsigned char cpbuf[sizeof(cudaGraphNodeParams)];
        memset(cpbuf, 0, sizeof(cpbuf));
        cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cpbuf);
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(P->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        P->enq = 0;
        enqueue_cycle(P, full, has_ref);
        k_cond<<<1, 1, 0, P->stream>>>(h, P->ndone, P->B, P->iters);
        P->enq += 1;
        cudaGraph_t outg = nullptr;
        cudaError_t ce = cudaStreamEndCapture(P->stream, &outg);
        if (ce != cudaSuccess) {
            cudaGraphDestroy(g);
            return fail(CMG_ECUDA, std::string("capture: ") + cudaGetErrorString(ce));
        }
    } else {
        CK(cudaStreamBeginCaptureToGraph(P->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        P->enq = 0;
        enqueue_cycle(P, full, has_ref);
        cudaGraph_t outg = nullptr;
        cudaError_t ce = cudaStreamEndCapture(P->stream, &outg);
        if (ce != cudaSuccess) {
            cudaGraphDestroy(g);
            return fail(CMG_ECUDA, std::string("capture: ") + cudaGetErrorString(ce));
        }
    }
    P->nodes_per_cycle = P->enq;
    cudaError_t ie = cudaGraphInstantiate(&P->exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(CMG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    P->gkey = key;
    return CMG_OK;
}

int ensure_trace(cmg_plan* P, int cap) {
    if (cap <= P->cap) return CMG_OK;
    for (int i = 0; i < 5; ++i) {
        if (P->tr[i]) cudaFree(P->tr[i]);
        P->tr[i] = nullptr;
    }
    for (int i = 0; i < 5; ++i) CK(cudaMalloc(&P->tr[i], sizeof(double) * (size_t)cap * P->B));
    P->cap = cap;
    // graphs embed the trace pointers -> rebuild
    if (P->exec) {
        cudaGraphExecDestroy(P->exec);
        P->exec = nullptr;
        P->gkey = -1;
    }
    return CMG_OK;
}

int check_cfg(double alpha, double eps, int max_outer, int inner, int stop_rule) {
    // SolverConfig.__post_init__ (driver.py:55-72)
    if (!(alpha > 0)) return fail(CMG_EINVAL, "alpha must be positive");
    if (!(eps > 0)) return fail(CMG_EINVAL, "epsilon must be positive");
    if (max_outer < 1) return fail(CMG_EINVAL, "max_outer must be at least 1");
    if (inner < 1 || inner > 15) return fail(CMG_EINVAL, "inner_iters must be in [1, 15]");
    if (stop_rule != 0 && stop_rule != 1) return fail(CMG_EINVAL, "stop_rule must be 'rel_energy' or 'rel_u'");
    return CMG_OK;
}

void fill_params(cmg_plan* P, SolveParams& sp, double alpha, double eps, int max_outer, int inner, int stop_rule,
                 bool has_ref, double peak) {
    memset(&sp, 0, sizeof(sp));
    sp.alpha = alpha;
    sp.half_alpha = 0.5 * alpha;  // tangent.py:340: 0.5 * alpha * sum
    sp.eps = eps;
    sp.peak = peak;
    sp.max_outer = max_outer;
    sp.inner = inner;
    sp.stop_rule = stop_rule;
    sp.has_ref = has_ref ? 1 : 0;
    sp.npix = P->N;
    for (int j = 1; j <= 6; ++j) {
        const double S = (double)(((1 << j) - 1) * ((1 << j) - 1));
        for (int t = 0; t < inner && t < 16; ++t) {
            const double eta = (t == 0) ? 1.0 : 1.0 / std::sqrt((double)t);  // fbs.py:68-72
            const double w = alpha * eta * S;                                 // fbs.py:89
            sp.w[j][t] = w;
            sp.den[j][t] = 2.0 + w;
        }
    }
}

template <typename T>
void enqueue_fpads(cmg_plan* P) {
    for (int j = 1; j <= P->layers; ++j) {
        Level& L = P->lv[j];
        if (L.general) enqueue_pad<T>(P, P->f, L.fpad, L.H, L.W, L.pstride, 1 + L.mp - P->m, 1 + L.np - P->n, false);
    }
}

int set_device(cmg_plan* P) {
    CK(cudaSetDevice(P->device));
    return CMG_OK;
}

int core_solve(cmg_plan* P, bool has_ref, double alpha, double eps, int max_outer, int inner, int stop_rule, int full,
               double peak, double* energy, double* rel_e, double* rel_u, double* psnr, double* seconds,
               int* iterations, int* status) {
    int rc = check_cfg(alpha, eps, max_outer, inner, stop_rule);
    if (rc) return rc;
    if (!(peak > 0)) return fail(CMG_EINVAL, "peak must be positive");
    rc = ensure_trace(P, max_outer + 1);
    if (rc) return rc;
    SolveParams sp;
    fill_params(P, sp, alpha, eps, max_outer, inner, stop_rule, has_ref, peak);
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemsetAsync(P->ndone, 0, sizeof(int) * 2, P->stream));
    rc = build_graph(P, full, has_ref);
    if (rc) return rc;
    CK(cudaEventRecord(P->e0, P->stream));
    P->enq = 0;
    const size_t bytes = P->esz * (size_t)P->N * P->B;
    CK(cudaMemcpyAsync(P->u, P->f, bytes, cudaMemcpyDeviceToDevice, P->stream));
    CK(cudaMemcpyAsync(P->uprev, P->f, bytes, cudaMemcpyDeviceToDevice, P->stream));
    if (P->dtype == CMG_F64) {
        enqueue_fpads<double>(P);
        enqueue_energy<double>(P, has_ref, nullptr, 1);
    } else {
        enqueue_fpads<float>(P);
        enqueue_energy<float>(P, has_ref, nullptr, 1);
    }
    CK(cudaGetLastError());
    const int init_launches = P->enq;
    int cycles = 0;
    if (P->use_while) {
        CK(cudaGraphLaunch(P->exec, P->stream));
        CK(cudaEventRecord(P->e1, P->stream));
        CK(cudaStreamSynchronize(P->stream));
        CK(cudaMemcpy(&cycles, P->iters, sizeof(int), cudaMemcpyDeviceToHost));
    } else {
        int chunk = 1, launched = 0;
        while (true) {
            const int c = std::min(chunk, max_outer - launched);
            for (int i = 0; i < c; ++i) CK(cudaGraphLaunch(P->exec, P->stream));
            launched += c;
            int nd = 0;
            CK(cudaMemcpyAsync(&nd, P->ndone, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
            CK(cudaStreamSynchronize(P->stream));
            if (nd >= P->B || launched >= max_outer) break;
            chunk = std::min(chunk * 2, 16);
        }
        CK(cudaEventRecord(P->e1, P->stream));
        CK(cudaStreamSynchronize(P->stream));
        cycles = launched;
    }
    CK(cudaEventElapsedTime(&P->dev_ms, P->e0, P->e1));
    P->cycles_run = cycles;
    P->launches = (long long)init_launches + (long long)cycles * P->nodes_per_cycle;
    std::vector<ImgState> hs(P->B);
    CK(cudaMemcpy(hs.data(), P->st, sizeof(ImgState) * P->B, cudaMemcpyDeviceToHost));
    double* outs[5] = {energy, rel_e, rel_u, psnr, seconds};
    for (int i = 0; i < 5; ++i) {
        if (!outs[i]) continue;
        const int cap = max_outer + 1;
        if (cap == P->cap) {
            CK(cudaMemcpy(outs[i], P->tr[i], sizeof(double) * (size_t)cap * P->B, cudaMemcpyDeviceToHost));
        } else {
            CK(cudaMemcpy2D(outs[i], sizeof(double) * cap, P->tr[i], sizeof(double) * P->cap, sizeof(double) * cap,
                            P->B, cudaMemcpyDeviceToHost));
        }
    }
    int overall = CMG_OK;
    for (int b = 0; b < P->B; ++b) {
        int s = hs[b].status;
        int it = hs[b].cycle;
        if (s == ST_RUNNING) s = ST_NOT_CONVERGED;  // defensive
        if (iterations) iterations[b] = it;
        if (status) status[b] = s;
        if (s != CMG_OK && overall == CMG_OK) overall = s;
    }
    if (overall == CMG_DIVERGED) g_err = "objective became non-finite";
    if (overall == CMG_ENONFINITE) g_err = "corrections must be finite";
    return overall;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int cmg_version(void) { return 100; }

const char* cmg_last_error(void) { return g_err.c_str(); }

int cmg_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        if (count) *count = 0;
        return fail(CMG_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    if (count) *count = c;
    return CMG_OK;
}

int cmg_plan_destroy(cmg_plan* P) {
    if (!P) return CMG_OK;
    cudaSetDevice(P->device);
    if (P->stream) cudaStreamSynchronize(P->stream);
    if (P->exec) cudaGraphExecDestroy(P->exec);
    void* ptrs[] = {P->u, P->uprev, P->f, P->ref, P->upad, P->epad, P->partials, P->st, P->ndone, P->eonly, P->P};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 5; ++i)
        if (P->tr[i]) cudaFree(P->tr[i]);
    for (int j = 1; j <= 6; ++j)
        if (P->lv[j].fpad) cudaFree(P->lv[j].fpad);
    if (P->e0) cudaEventDestroy(P->e0);
    if (P->e1) cudaEventDestroy(P->e1);
    if (P->stream) cudaStreamDestroy(P->stream);
    delete P;
    return CMG_OK;
}

int cmg_plan_create(cmg_plan** out, int m, int n, int batch, int layers, int mode, int dtype, int precision,
                    int device) {
    if (!out) return fail(CMG_EINVAL, "out is NULL");
    *out = nullptr;
    if (m < 1 || n < 1) return fail(CMG_EINVAL, "image dimensions must be positive");
    if (batch < 1) return fail(CMG_EINVAL, "batch must be positive");
    if (layers < 1 || layers > 6) return fail(CMG_EINVAL, "layers must be in [1, 6]");
    if (mode != CMG_MODE_MEAN && mode != CMG_MODE_GAUSS)
        return fail(CMG_EINVAL, "mode must be 'mean' or 'gaussian'");
    if (dtype != CMG_F64 && dtype != CMG_F32) return fail(CMG_EINVAL, "dtype must be f64 or f32");
    if (precision != CMG_PREC_EXACT && precision != CMG_PREC_FAST) return fail(CMG_EINVAL, "bad precision");
    if ((long long)m * n > (1LL << 31)) return fail(CMG_EINVAL, "image too large (m*n must be < 2^31)");
    cmg_plan* P = new cmg_plan();
    P->m = m;
    P->n = n;
    P->B = batch;
    P->layers = layers;
    P->mode = mode;
    P->dtype = dtype;
    P->prec = (mode == CMG_MODE_GAUSS) ? CMG_PREC_EXACT : precision;
    P->device = device;
    P->esz = dtype == CMG_F64 ? 8 : 4;
    P->N = (long long)m * n;
    const char* nw = getenv("CMG_NO_WHILE");
    P->use_while = !(nw && nw[0] == '1');
    auto bail = [&](int rc) {
        cmg_plan_destroy(P);
        return rc;
    };
#define CKP(x)                                                                                               \
    do {                                                                                                     \
        cudaError_t e_ = (x);                                                                                \
        if (e_ != cudaSuccess) return bail(fail(CMG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_))); \
    } while (0)
    CKP(cudaSetDevice(device));
    CKP(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
    CKP(cudaEventCreate(&P->e0));
    CKP(cudaEventCreate(&P->e1));
    const size_t bytes = P->esz * (size_t)P->N * batch;
    CKP(cudaMalloc(&P->u, bytes));
    CKP(cudaMalloc(&P->uprev, bytes));
    CKP(cudaMalloc(&P->f, bytes));
    size_t maxpad = 0;
    for (int j = 1; j <= layers; ++j) {
        Level& L = P->lv[j];
        L.layer = j;
        L.s = (1 << j) - 1;
        L.r = 1 << (j - 1);
        L.mj = (m + L.s - 1) / L.s;
        L.nj = (n + L.s - 1) / L.s;
        L.mp = L.mj * L.s;
        L.np = L.nj * L.s;
        L.general = !(single_chunk(m, 1 + L.mp - m) && single_chunk(n, 1 + L.np - n));
        L.H = L.mp + 2;
        L.W = L.np + 2;
        L.pstride = (long long)L.H * L.W;
        if (L.general) {
            CKP(cudaMalloc(&L.fpad, P->esz * (size_t)L.pstride * batch));
            maxpad = std::max(maxpad, (size_t)L.pstride);
        }
    }
    if (maxpad) {
        CKP(cudaMalloc(&P->upad, P->esz * maxpad * batch));
        P->upad_elems = maxpad;
    }
    P->egeneral = !(single_chunk(m, 1) && single_chunk(n, 1));
    P->eH = m + 2;
    P->eW = n + 2;
    P->epstride = (long long)P->eH * P->eW;
    if (P->egeneral) CKP(cudaMalloc(&P->epad, P->esz * (size_t)P->epstride * batch));
    long long want = std::max(1, 1184 / batch);
    P->nbx = (int)std::max(1LL, std::min(want, (P->N + 255) / 256));
    CKP(cudaMalloc(&P->partials, sizeof(double) * NSUM * (size_t)P->nbx * batch));
    CKP(cudaMalloc(&P->st, sizeof(ImgState) * batch));
    CKP(cudaMalloc(&P->ndone, sizeof(int) * 2));
    P->iters = P->ndone + 1;
    CKP(cudaMalloc(&P->eonly, sizeof(double) * batch));
    CKP(cudaMalloc(&P->P, sizeof(SolveParams)));
#undef CKP
    *out = P;
    return CMG_OK;
}

int cmg_solve_device(cmg_plan* P, const void* f_dev, const void* ref_dev, void* u_dev_out, double alpha,
                     double epsilon, int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak,
                     double* energy, double* rel_energy, double* rel_u, double* psnr, double* seconds,
                     int* iterations, int* status) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    int rc = set_device(P);
    if (rc) return rc;
    const size_t bytes = P->esz * (size_t)P->N * P->B;
    if (f_dev && f_dev != P->f) CK(cudaMemcpyAsync(P->f, f_dev, bytes, cudaMemcpyDeviceToDevice, P->stream));
    if (ref_dev) {
        if (!P->ref) CK(cudaMalloc(&P->ref, bytes));
        if (ref_dev != P->ref) CK(cudaMemcpyAsync(P->ref, ref_dev, bytes, cudaMemcpyDeviceToDevice, P->stream));
    }
    rc = core_solve(P, ref_dev != nullptr, alpha, epsilon, max_outer, inner_iters, stop_rule, full_vcycle, peak,
                    energy, rel_energy, rel_u, psnr, seconds, iterations, status);
    if (rc == CMG_EINVAL || rc == CMG_ECUDA) return rc;
    if (u_dev_out && u_dev_out != P->u) {
        CK(cudaMemcpyAsync(u_dev_out, P->u, bytes, cudaMemcpyDeviceToDevice, P->stream));
        CK(cudaStreamSynchronize(P->stream));
    }
    return rc;
}

int cmg_solve(cmg_plan* P, const void* f_host, const void* ref_host, void* u_host_out, double alpha, double epsilon,
              int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak, double* energy,
              double* rel_energy, double* rel_u, double* psnr, double* seconds, int* iterations, int* status) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    if (!f_host) return fail(CMG_EINVAL, "f is NULL");
    int rc = set_device(P);
    if (rc) return rc;
    const size_t bytes = P->esz * (size_t)P->N * P->B;
    CK(cudaMemcpyAsync(P->f, f_host, bytes, cudaMemcpyHostToDevice, P->stream));
    if (ref_host) {
        if (!P->ref) CK(cudaMalloc(&P->ref, bytes));
        CK(cudaMemcpyAsync(P->ref, ref_host, bytes, cudaMemcpyHostToDevice, P->stream));
    }
    rc = core_solve(P, ref_host != nullptr, alpha, epsilon, max_outer, inner_iters, stop_rule, full_vcycle, peak,
                    energy, rel_energy, rel_u, psnr, seconds, iterations, status);
    if (rc == CMG_EINVAL || rc == CMG_ECUDA) return rc;
    if (u_host_out) {
        CK(cudaMemcpyAsync(u_host_out, P->u, bytes, cudaMemcpyDeviceToHost, P->stream));
        CK(cudaStreamSynchronize(P->stream));
    }
    return rc;
}

int cmg_sweep_layer(cmg_plan* P, void* u_host, const void* f_host, int layer, double alpha, int inner_iters) {
    if (!P || !u_host || !f_host) return fail(CMG_EINVAL, "NULL argument");
    if (layer < 1 || layer > P->layers) return fail(CMG_EINVAL, "layer outside the plan's hierarchy");
    int rc = check_cfg(alpha, 1.0, 1, inner_iters, 0);
    if (rc) return rc;
    rc = set_device(P);
    if (rc) return rc;
    const size_t bytes = P->esz * (size_t)P->N * P->B;
    SolveParams sp;
    fill_params(P, sp, alpha, 1.0, 1, inner_iters, 0, false, 1.0);
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemcpyAsync(P->u, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->f, f_host, bytes, cudaMemcpyHostToDevice, P->stream));
    if (P->dtype == CMG_F64) {
        enqueue_fpads<double>(P);
        for (int c = 0; c < 4; ++c) enqueue_sweep<double>(P, layer, c);
    } else {
        enqueue_fpads<float>(P);
        for (int c = 0; c < 4; ++c) enqueue_sweep<float>(P, layer, c);
    }
    CK(cudaGetLastError());
    std::vector<ImgState> hs(P->B);
    CK(cudaMemcpyAsync(hs.data(), P->st, sizeof(ImgState) * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaMemcpyAsync(u_host, P->u, bytes, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    for (int b = 0; b < P->B; ++b)
        if (hs[b].bad) return fail(CMG_ENONFINITE, "corrections must be finite");
    return CMG_OK;
}

int cmg_energy(cmg_plan* P, const void* u_host, const void* f_host, double alpha, double* energy_out) {
    if (!P || !u_host || !f_host || !energy_out) return fail(CMG_EINVAL, "NULL argument");
    if (!(alpha > 0)) return fail(CMG_EINVAL, "alpha must be positive");
    int rc = set_device(P);
    if (rc) return rc;
    const size_t bytes = P->esz * (size_t)P->N * P->B;
    SolveParams sp;
    fill_params(P, sp, alpha, 1.0, 1, 1, 0, false, 1.0);
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemcpyAsync(P->u, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->uprev, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->f, f_host, bytes, cudaMemcpyHostToDevice, P->stream));
    if (P->dtype == CMG_F64)
        enqueue_energy<double>(P, false, P->eonly, 0);
    else
        enqueue_energy<float>(P, false, P->eonly, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(energy_out, P->eonly, sizeof(double) * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

int cmg_plane_table(int layer, int* offsets, double* ds2) {
    if (layer < 1 || layer > 6) return fail(-1, "layer must be in [1, 6]");
    const int cnt = 1 << (layer + 2);
    for (int i = 0; i < cnt; ++i) {
        for (int k = 0; k < 6; ++k)
            if (offsets) offsets[6 * i + k] = kCmgPlaneOff[i][k];
        if (ds2) ds2[i] = (double)(kCmgPlaneOff[i][0] * kCmgPlaneOff[i][0] + kCmgPlaneOff[i][1] * kCmgPlaneOff[i][1]);
    }
    return cnt;
}

int cmg_plan_stats(cmg_plan* P, long long* kernel_launches, int* cycles_run, double* device_ms) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    if (kernel_launches) *kernel_launches = P->launches;
    if (cycles_run) *cycles_run = P->cycles_run;
    if (device_ms) *device_ms = P->dev_ms;
    return CMG_OK;
}

int cmg_time_sweep(cmg_plan* P, int layer, int color, int reps, double* ms_per_launch) {
    if (!P || !ms_per_launch) return fail(CMG_EINVAL, "NULL argument");
    if (layer < 1 || layer > P->layers || color > 3 || reps < 1) return fail(CMG_EINVAL, "bad arguments");
    int rc = set_device(P);
    if (rc) return rc;
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    auto one = [&]() {
        for (int c = (color < 0 ? 0 : color); c <= (color < 0 ? 3 : color); ++c) {
            if (P->dtype == CMG_F64)
                enqueue_sweep<double>(P, layer, c);
            else
                enqueue_sweep<float>(P, layer, c);
        }
    };
    one();  // warm-up
    CK(cudaEventRecord(P->e0, P->stream));
    for (int i = 0; i < reps; ++i) one();
    CK(cudaEventRecord(P->e1, P->stream));
    CK(cudaEventSynchronize(P->e1));
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, P->e0, P->e1));
    *ms_per_launch = (double)ms / reps;
    return CMG_OK;
}

void* cmg_host_alloc(unsigned long long bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
        g_err = "cudaMallocHost failed";
        return nullptr;
    }
    return p;
}

int cmg_host_free(void* p) {
    if (p) CK(cudaFreeHost(p));
    return CMG_OK;
}

}  // extern "C"
