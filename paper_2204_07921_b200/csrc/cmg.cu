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
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are no-ops unless a profiler is attached

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cmg.h"
#include "cmg_plan.h"
#include "cmg_metrics.cuh"

// NVTX range of one C-ABI call (shows up in Nsight Systems / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

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

inline bool single_chunk(int len, int pad_after) { return len >= 2 && pad_after <= len - 1; }

}  // namespace

namespace cmg {
// error reporting for the other translation units (cmg_recon.cu)
int set_error(int code, const char* msg) {
    g_err = msg;
    return code;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_tmap(CUtensorMap* out, const void* base, int esz, int m, int n, int B, int boxcode) {
    const int box = boxcode / 4096, boxh = boxcode % 4096;
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = (EncodeTiledFn)p;
    }
    if (((long long)n * esz) % 16 != 0 || ((long long)box * esz) % 16 != 0 || box > 256 || boxh > 256) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, (cuuint64_t)B};
    const cuuint64_t strides[2] = {(cuuint64_t)n * esz, (cuuint64_t)m * n * esz};
    const cuuint32_t boxd[3] = {(cuuint32_t)box, (cuuint32_t)boxh, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(out, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<void*>(base), dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace cmg

namespace {

__global__ void k_cond(cudaGraphConditionalHandle h, const int* ndone, int B, int* iters) {
    cmg::pdl_sync();
    *iters += 1;
    cudaGraphSetConditional(h, (*ndone < B) ? 1u : 0u);
}

// L2 bandwidth probe: every thread streams 16-byte words, `reps` passes
__global__ void k_l2_read(const uint4* __restrict__ buf, long long n16, int reps, unsigned* sink) {
    unsigned acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldcg(buf + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x9e3779b9u) sink[(blockIdx.x * blockDim.x + threadIdx.x) & 1048575] = acc;
}

// FP64 pipe probe: ILP independent chains of dependent DFMAs per thread
template <int ILP>
__global__ void k_fp64_chain(double* out, int iters, double a, double b, long long* cycles) {
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = (double)(threadIdx.x + j) * 1e-3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = __fma_rn(x[j], a, b);
    }
    const long long t1 = clock64();
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) sum += x[j];
    if (sum == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
    if (cycles && blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
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
    enqueue_copy_prev<T>(P);
    for (int j : layer_sequence(P->layers, full))
        for (int c = 0; c < 4; ++c) enqueue_sweep<T>(P, j, c);
    enqueue_energy<T>(P, has_ref, nullptr, 0);
}

void enqueue_cycle(cmg_plan* P, int full, bool has_ref) {
    if (P->efuse) {
        if (P->dtype == CMG_F64)
            enqueue_body_efused<double>(P, full, has_ref);
        else
            enqueue_body_efused<float>(P, full, has_ref);
        return;
    }
    if (P->fused) {
        if (P->dtype == CMG_F64)
            enqueue_body_fused<double>(P, full, has_ref);
        else
            enqueue_body_fused<float>(P, full, has_ref);
        return;
    }
    if (P->dtype == CMG_F64)
        enqueue_cycle_T<double>(P, full, has_ref);
    else
        enqueue_cycle_T<float>(P, full, has_ref);
}

int build_graph(cmg_plan* P, int full, bool has_ref) {
    const int key = full * 2 + (has_ref ? 1 : 0);
    // kernel arguments carry the backward-step constants: rebuild when they change
    if (P->exec && P->gkey == key && P->galpha == P->hostP.alpha && P->ginner == P->hostP.inner) return CMG_OK;
    P->galpha = P->hostP.alpha;
    P->ginner = P->hostP.inner;
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
        P->cur_cond = P->fused_finalize ? (unsigned long long)h : 0ULL;
        enqueue_cycle(P, full, has_ref);
        P->cur_cond = 0;
        if (!P->fused_finalize) {
            k_cond<<<1, 1, 0, P->stream>>>(h, P->ndone, P->B, P->iters);
            P->enq += 1;
            stamp(P, 99);
        }
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
    if (P->launch_err != cudaSuccess) {
        const cudaError_t le = P->launch_err;
        P->launch_err = cudaSuccess;
        cudaGraphDestroy(g);
        return fail(CMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(le));
    }
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

// one level visit in_index -> out_index on the plan stream (strip steps):
// the fused tile / row-parity kernel, or a copy + the in-place colour sweeps
void enqueue_level(cmg_plan* P, int layer, int in_index, int out_index) {
    const bool fusedj = P->fused && layer <= 3 && ((P->fuse_mask >> (layer - 1)) & 1);
    if (fusedj) {
        if (P->dtype == CMG_F64)
            enqueue_fused_level<double>(P, layer, P->ubuf[in_index], P->ubuf[out_index]);
        else
            enqueue_fused_level<float>(P, layer, P->ubuf[in_index], P->ubuf[out_index]);
        return;
    }
    cudaMemcpyAsync(P->ubuf[out_index], P->ubuf[in_index], P->esz * (size_t)P->N * P->B, cudaMemcpyDeviceToDevice,
                    P->stream);
    void* save = P->u;
    P->u = P->ubuf[out_index];
    for (int c = 0; c < 4; ++c) {
        if (P->dtype == CMG_F64)
            enqueue_sweep<double>(P, layer, c);
        else
            enqueue_sweep<float>(P, layer, c);
    }
    P->u = save;
}

// strip mode: per-image non-finite-correction flag next to the 5 energy sums
__global__ void k_strip_flags(const ImgState* st, double* raw6, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) raw6[(long long)B * NSUM + b] = st[b].bad ? 1.0 : 0.0;
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

int set_device(cmg_plan* P) {
    CK(cudaSetDevice(P->device));
    return CMG_OK;
}

int core_solve(cmg_plan* P, bool has_ref, double alpha, double eps, int max_outer, int inner, int stop_rule, int full,
               double peak, double* energy, double* rel_e, double* rel_u, double* psnr, double* seconds,
               int* iterations, int* status) {
    NvtxRange nvtx("cmg core_solve (V-cycle graph)");
    int rc = check_cfg(alpha, eps, max_outer, inner, stop_rule);
    if (rc) return rc;
    if (!(peak > 0)) return fail(CMG_EINVAL, "peak must be positive");
    rc = ensure_trace(P, max_outer + 1);
    if (rc) return rc;
    SolveParams sp;
    fill_params(P, sp, alpha, eps, max_outer, inner, stop_rule, has_ref, peak);
    P->hostP = sp;
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemsetAsync(P->ndone, 0, sizeof(int) * 2, P->stream));
    int cycles = 0, bodies = 0, init_launches = 0;
    {
        if (!P->no_graph) {
            rc = build_graph(P, full, has_ref);
            if (rc) return rc;
        }
        CK(cudaEventRecord(P->e0, P->stream));
        P->enq = 0;
        const size_t bytes = P->esz * (size_t)P->N * P->B;
        CK(cudaMemcpyAsync(P->u, P->f, bytes, cudaMemcpyDeviceToDevice, P->stream));
        if (!P->fused) CK(cudaMemcpyAsync(P->uprev, P->f, bytes, cudaMemcpyDeviceToDevice, P->stream));
        // initial energy (cycle 0): a separate pass, or the first level-1 kernel of the
        // energy-fused body
        if (P->dtype == CMG_F64) {
            enqueue_fpads<double>(P);
            enqueue_fsums<double>(P);
            if (!P->efuse)
                enqueue_energy_ptrs<double>(P, P->u, P->fused ? P->u : P->uprev, has_ref, nullptr, 1, nullptr, 0, -1);
        } else {
            enqueue_fpads<float>(P);
            enqueue_fsums<float>(P);
            if (!P->efuse)
                enqueue_energy_ptrs<float>(P, P->u, P->fused ? P->u : P->uprev, has_ref, nullptr, 1, nullptr, 0, -1);
        }
        CK(cudaGetLastError());
        if (P->launch_err != cudaSuccess) {
            const cudaError_t le = P->launch_err;
            P->launch_err = cudaSuccess;
            return fail(CMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(le));
        }
        init_launches = P->enq;
        if (P->use_while) {
            CK(cudaGraphLaunch(P->exec, P->stream));
            if (P->fused) {  // stopped images whose final u is not in buffer 0
                if (P->dtype == CMG_F64)
                    enqueue_collect<double>(P);
                else
                    enqueue_collect<float>(P);
            }
            CK(cudaEventRecord(P->e1, P->stream));
            CK(cudaStreamSynchronize(P->stream));
            bodies = -1;  // counted from the per-image cycle counters below
        } else {
            int chunk = 1, launched = 0;
            // cycles per body; the energy-fused body needs one more level-1 visit (the
            // energy of the last cycle is computed by the next cycle's level-1 kernel)
            const int per = P->efuse ? efused_cycles_per_body(P, full) : (P->fused ? 2 : 1);
            const int maxb = (max_outer + (P->efuse ? 1 : 0) + per - 1) / per;
            while (true) {
                const int c = std::min(chunk, maxb - launched);
                for (int i = 0; i < c; ++i) {
                    if (P->no_graph) {  // profiling mode: plain stream launches, same kernels
                        const int e0 = P->enq;
                        enqueue_cycle(P, full, has_ref);
                        P->nodes_per_cycle = P->enq - e0;
                        CK(cudaGetLastError());
                    } else {
                        CK(cudaGraphLaunch(P->exec, P->stream));
                    }
                }
                launched += c;
                int nd = 0;
                CK(cudaMemcpyAsync(&nd, P->ndone, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
                CK(cudaStreamSynchronize(P->stream));
                if (nd >= P->B || launched >= maxb) break;
                chunk = std::min(chunk * 2, 16);
            }
            if (P->fused) {
                if (P->dtype == CMG_F64)
                    enqueue_collect<double>(P);
                else
                    enqueue_collect<float>(P);
            }
            CK(cudaEventRecord(P->e1, P->stream));
            CK(cudaStreamSynchronize(P->stream));
            bodies = launched;
        }
    }
    CK(cudaEventElapsedTime(&P->dev_ms, P->e0, P->e1));
    std::vector<ImgState> hs(P->B);
    CK(cudaMemcpy(hs.data(), P->st, sizeof(ImgState) * P->B, cudaMemcpyDeviceToHost));
    {
        cycles = 0;
        for (int b = 0; b < P->B; ++b)
            cycles = std::max(cycles, hs[b].cycle + ((hs[b].status == ST_DIVERGED || hs[b].status == ST_NONFINITE) ? 1 : 0));
    }
    P->cycles_run = cycles;
    {
        // kernels executed on the device: set-up kernels + every kernel node of
        // every WHILE-body replay (a body holds 2 cycles on the fused path)
        const int per = P->efuse ? efused_cycles_per_body(P, full) : (P->fused ? 2 : 1);
        if (bodies < 0) bodies = std::max(1, (cycles + (P->efuse ? 1 : 0) + per - 1) / per);
        P->launches = (long long)init_launches + (long long)bodies * P->nodes_per_cycle + (P->fused ? 1 : 0);
    }
    if (P->stamps) {
        std::vector<unsigned long long> sb(P->stamps_cap);
        CK(cudaMemcpy(sb.data(), P->stamps, sizeof(unsigned long long) * P->stamps_cap, cudaMemcpyDeviceToHost));
        const int cnt = std::min((int)(sb[0] & 0xffffffffu), P->stamps_cap - 1);
        FILE* fo = fopen(getenv("CMG_STAMPS_FILE") ? getenv("CMG_STAMPS_FILE") : "cmg_stamps.txt", "w");
        if (fo) {
            for (int i = 0; i < cnt; ++i) fprintf(fo, "%d %llu\n", (int)(sb[1 + i] & 0xff), sb[1 + i] >> 8);
            fclose(fo);
        }
        CK(cudaMemset(P->stamps, 0, sizeof(unsigned long long) * P->stamps_cap));
    }
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
    void* ptrs[] = {P->u, P->uprev, P->ubuf[2], P->f, P->ref, P->upad, P->epad, P->partials, P->st, P->ndone, P->eonly, P->raw5, P->P, P->stamps, P->tickets, P->fsum[2], P->fsum[3]};
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
    if (const char* ng = getenv("CMG_NO_GRAPH")) {
        P->no_graph = ng[0] == '1';
        if (P->no_graph) P->use_while = false;
    }
    if (const char* t2 = getenv("CMG_TS2")) P->ts2 = atoi(t2);
    if (const char* t3 = getenv("CMG_TS3")) P->ts3 = atoi(t3);
    {
        // level 1 always runs as one fused tile kernel; levels 2-3 only when the
        // image is large enough that the fused SMEM tiles fill the GPU several
        // times over (small images are latency-bound: per-colour team kernels win)
        const int tp2 = dtype == CMG_F64 ? 16 : 32, tp3 = dtype == CMG_F64 ? 4 : 8;
        // (per-image tile grids must also be large: border tiles cannot use TMA)
        auto tiles = [&](int s, int tp) {
            const long long mj = (m + s - 1) / s, nj = (n + s - 1) / s;
            return ((mj + tp - 1) / tp) * ((nj + tp - 1) / tp);
        };
        P->fuse_mask = 1;
        if (layers >= 2 && tiles(3, tp2) >= 400 && tiles(3, tp2) * batch >= 2048) P->fuse_mask |= 2;
        // level 3: the per-colour team kernels beat the fused tile at every size
        // measured (16384^2 fp32: 1.80 vs 2.92 ms; the tile recomputes ~2x the
        // patches and holds 84 KB of shared memory per CTA), so it stays opt-in
        (void)tp3;
        // large fp32 fast jobs are throughput-bound: 8-lane teams (16384^2: 1.80
        // vs 2.26 ms); small ones latency-bound, and fp64 exact prefers 16 lanes
        // at every size (2048^2: 96 vs 266 us)
        if (dtype == CMG_F32 && P->prec == CMG_PREC_FAST && (long long)batch * m * n >= (4LL << 20) &&
            !getenv("CMG_TS3"))
            P->ts3 = 8;
    }
    // levels 2-3 as two row-parity launches each (k_rowpair): half the launches and
    // half the traffic of four colour launches; they join the fused X -> Y rotation
    // measured (B200, round 1): a win for latency-bound jobs (1024^2 fp64 fast: 4.13 -> 3.80 ms
    // per solve), a loss for large throughput-bound jobs (16384^2 level 2:
    // 3.6 vs 1.3 ms with the coarse tile), where the per-colour / tile kernels stay
    const bool small_job = (long long)batch * m * n < (4LL << 20);
    // (bench, config 3: fp64 exact 5.24 ms with 8-lane level-2 teams vs 5.04 ms with 4;
    // fp64 fast 3.92 vs 3.75; configs 1 / 2: 2.69 -> 2.61 ms, 18.7 -> 18.1 ms with row pairs)
    P->rowpair = small_job ? 3 : 0;
    P->rp_ts2 = 4;
    // large fast-mean jobs: level 3 as row-parity launches with one thread per
    // patch (per-patch f sums, u-only windows): one read and one write of u per
    // level instead of four per-colour passes
    const bool fast_mean = mode == CMG_MODE_MEAN && P->prec == CMG_PREC_FAST;
    // (B200, round 2: 16384^2 level 3 1.37 -> 0.44 ms, level 2 0.89 -> 0.65 ms vs the
    // fused coarse tile; 64 x 512^2 level 2 133 -> 87 us with 32-thread CTAs.  Level 3
    // only on wide images: a 512-wide image leaves most of the window empty and
    // config 4 keeps the per-colour team kernels there, 111 vs 153 us)
    if (!small_job && fast_mean && layers >= 2 && n >= 256) {
        P->rowpair |= 1;
        P->rp1 |= 1;
    }
    if (!small_job && fast_mean && layers >= 3 && n >= 2048) {
        P->rowpair |= 2;
        P->rp1 |= 2;
    }
    P->rp_nt = n >= 2048 ? 64 : 32;
    P->rp_nt2 = (n < 2048 && (n + 2) / 3 <= 172) ? 172 : 0;
    if (const char* rp = getenv("CMG_ROWPAIR")) P->rowpair = atoi(rp) & 3;
    if (const char* r1 = getenv("CMG_RP1")) P->rp1 = atoi(r1) & 3;
    if (const char* rb = getenv("CMG_RP_BULK")) P->rp_bulk = atoi(rb);
    if (const char* rt = getenv("CMG_RP_TMA")) P->rp_tma = atoi(rt);
    if (const char* rn = getenv("CMG_RP_NT")) P->rp_nt = atoi(rn);
    if (const char* rn = getenv("CMG_RP_NT2")) P->rp_nt2 = atoi(rn);
    if (const char* rs = getenv("CMG_RP_STAGES")) P->rp_stages = atoi(rs);
    if (const char* rt = getenv("CMG_RP_TS2")) P->rp_ts2 = atoi(rt);
    if (layers >= 2 && (P->rowpair & 1)) P->fuse_mask |= 2;
    if (layers >= 3 && (P->rowpair & 2)) P->fuse_mask |= 4;
    if (const char* fm = getenv("CMG_FUSE_MASK")) P->fuse_mask = atoi(fm) | 1;
    if (const char* dg = getenv("CMG_DBG")) P->dbg = atoi(dg);
    if (const char* sp = getenv("CMG_STAMPS")) {
        if (atoi(sp) > 0) {
            P->stamps_cap = 1 << 16;
            if (cudaMalloc(&P->stamps, sizeof(unsigned long long) * P->stamps_cap) != cudaSuccess) {
                P->stamps = nullptr;
            } else {
                cudaMemset(P->stamps, 0, sizeof(unsigned long long) * P->stamps_cap);
            }
        }
    }
    // packed level-1 kernel: 56 x 120 tiles for large images (less halo per pixel,
    // 16384^2: 1.03 vs 1.11 ms), 56 x 56 otherwise (more CTAs for small images)
    // (f read from global memory by each pixel's own phase instead of staged:
    // half the shared memory, 5 instead of 3 CTAs per SM; 16384^2: 0.919 -> 0.879 ms)
    if ((long long)m * n >= (4LL << 20) && n >= 240) P->l1x2 = 11;
    if (const char* lx = getenv("CMG_L1X2")) P->l1x2 = atoi(lx);
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
    CKP(cudaMalloc(&P->ubuf[2], bytes));
    P->ubuf[0] = P->u;
    P->ubuf[1] = P->uprev;
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
    // per-patch f sums for the fast mean path of levels 2-3 (f* without f pixels)
    if (const char* fs = getenv("CMG_FSUM")) P->use_fsum = atoi(fs) != 0;
    if (P->use_fsum && mode == CMG_MODE_MEAN && P->prec == CMG_PREC_FAST)
        for (int j = 2; j <= std::min(layers, 3); ++j)
            if (!P->lv[j].general)
                CKP(cudaMalloc(&P->fsum[j], sizeof(double) * (size_t)P->lv[j].mj * P->lv[j].nj * batch));
    P->egeneral = !(single_chunk(m, 1) && single_chunk(n, 1));
    P->eH = m + 2;
    P->eW = n + 2;
    P->epstride = (long long)P->eH * P->eW;
    if (P->egeneral) CKP(cudaMalloc(&P->epad, P->esz * (size_t)P->epstride * batch));
    {
        bool gen = P->egeneral;
        for (int j = 1; j <= layers; ++j) gen = gen || P->lv[j].general;
        bool fgen = false;
        for (int j = 1; j <= std::min(layers, 3); ++j) fgen = fgen || P->lv[j].general;
        const char* fe = getenv("CMG_FUSED");
        P->fused = !fgen && !(fe && fe[0] == '0');
        (void)gen;
    }
    {
        const char* te = getenv("CMG_TMA");
        const int tmode = te ? atoi(te) : 1;  // 0 off, 1 levels 2-3, 2 / 3 only that level
        const bool allow = tmode != 0;
        for (int j = 2; j <= std::min(layers, 3) && allow; ++j) {
            if (tmode >= 2 && j != tmode) continue;
            const int box = (dtype == CMG_F64) ? coarse_region<double>(j) : coarse_region<float>(j);
            bool ok = true;
            for (int bi = 0; bi < 4 && ok; ++bi)
                ok = make_tmap(&P->tmap[j][bi], bi < 3 ? P->ubuf[bi] : P->f, (int)P->esz, m, n, batch, box);
            P->tma_ok[j] = ok;
        }
    }
    // energy CTAs per image: row bands of >= 4 rows, ~1184 CTAs in total
    long long want = std::max(1, 1184 / batch);
    if (const char* nb = getenv("CMG_ENERGY_CTAS")) want = std::max(1, atoi(nb) / batch);
    P->nbx = (int)std::max(1LL, std::min(want, (long long)(m + 3) / 4));
    if (const char* et = getenv("CMG_ENERGY_TARGET")) {
        // opt-in 2-D grid (row bands x 256-column chunks, one column per thread).  Measured
        // at 1024^2 (B200): 21 us at 256 CTAs, 28 us at 1024, 37 us at 2048 vs 19.8 us for
        // the default 256 full-width bands -- the per-CTA ticket atomics and the longer
        // finalize outweigh the shorter per-thread chains
        P->ncb = (int)((n + 255) / 256);
        const long long target = std::max(1, atoi(et));
        const long long nrb = std::max(1LL, std::min<long long>((target + batch * P->ncb - 1) / (batch * P->ncb),
                                                                (m + 1) / 2));
        P->nbx = (int)(nrb * P->ncb);
    }
    // rows streamed by bulk async copies (k_energy_bulk): 16-byte aligned rows
    {
        const char* eb = getenv("CMG_EBULK");
        // large jobs only: below ~4M pixels the pass is latency-bound and the
        // row-band kernel (no pipeline fill) is faster
        const bool big = (long long)batch * m * n >= (4LL << 20);
        const bool on = (eb ? atoi(eb) != 0 : big) && !P->egeneral && ((size_t)n * P->esz) % 16 == 0;
        if (on) {
            if (dtype == CMG_F32)
                P->eb_px = n > 512 ? 4 : (n > 256 ? 2 : 1);
            else
                P->eb_px = n > 256 ? 2 : 1;
            if (const char* ns = getenv("CMG_EBULK_NS")) P->eb_ns = std::min(8, std::max(2, atoi(ns)));
            const int nb = dtype == CMG_F64 ? energy_bulk_cfg<double>(batch, m, n, P->eb_px, P->eb_ns, &P->eb_H)
                                            : energy_bulk_cfg<float>(batch, m, n, P->eb_px, P->eb_ns, &P->eb_H);
            if (!getenv("CMG_ENERGY_CTAS")) P->nbx = nb;
            P->ncb = 1;
        }
    }
    if (getenv("CMG_VERBOSE"))
        fprintf(stderr, "cmg plan %dx%dx%d: energy CTAs/image %d (bulk px %d ns %d H %d), fused L2 %d L3 %d\n", m,
                n, batch, P->nbx, P->eb_px, P->eb_ns, P->eb_H, (P->fuse_mask >> 1) & 1, (P->fuse_mask >> 2) & 1);
    if (const char* ff = getenv("CMG_FUSED_FINALIZE")) P->fused_finalize = atoi(ff) != 0;
    // energy-fused cycles: the level-1 tile kernel (k_l1_tile; fp32 fast mean keeps the
    // packed k_l1_x2 kernel and the separate bulk energy pass) sums the energy of its
    // input; partials per level-1 CTA (tiles >= 32 x 32)
    {
        // packed fp32 level-1 kernel (k_l1_x2): only for latency-bound (small) jobs; on
        // large ones the issue-heavy packed kernel pays more for the energy terms than the
        // streamlined bulk energy pass costs (16384^2: 2.06 ms vs 0.90 + 0.56 ms)
        const bool x2 = dtype == CMG_F32 && P->prec == CMG_PREC_FAST && mode == CMG_MODE_MEAN && P->l1x2;
        P->efuse = P->fused && P->fused_finalize && (!x2 || small_job);
        if (const char* ef = getenv("CMG_EFUSE")) P->efuse = P->efuse && atoi(ef) != 0;
    }
    const long long l1tiles = (long long)((m + 27) / 28) * ((n + 31) / 32);  // covers 28-row tiles too
    const long long nparts = std::max<long long>(P->nbx, P->efuse ? l1tiles : 0);
    CKP(cudaMalloc(&P->partials, sizeof(double) * NSUM * (size_t)nparts * batch));
    P->pcap = (int)(nparts * batch);
    CKP(cudaMalloc(&P->st, sizeof(ImgState) * batch));
    CKP(cudaMalloc(&P->ndone, sizeof(int) * 2));
    P->iters = P->ndone + 1;
    CKP(cudaMalloc(&P->eonly, sizeof(double) * batch));
    CKP(cudaMalloc(&P->raw5, sizeof(double) * (NSUM + 1) * batch));  // strip mode: 5 sums + flag per image
    CKP(cudaMalloc(&P->tickets, sizeof(int) * (batch + 1)));
    CKP(cudaMemset(P->tickets, 0, sizeof(int) * (batch + 1)));
    if (const char* pd = getenv("CMG_PDL")) P->pdl = atoi(pd) != 0;
    // 32 x 64 level-1 tiles once they fill the GPU (1024^2 fp64 exact: 48.7 -> 47.3 us,
    // 4096^2: 643 -> 579 us; 512^2 has too few: 20.3 -> 27.2 us)
    P->l1_wide = (long long)batch * m * n >= (1LL << 20);
    if (const char* lw = getenv("CMG_L1_WIDE")) P->l1_wide = atoi(lw) != 0;
    if (dtype == CMG_F64) {
        // fp64 level-1 tile shape: the kernel runs 4 CTAs of 256 threads per SM and its
        // duration is that of the fullest SM, so pick the shape with the least
        // (CTA waves) x (pixels a CTA relaxes, halo included).  1024^2: 28 x 64 tiles
        // = 37 x 16 = 592 CTAs = exactly 4 per SM (level-1 sweep 45.6 -> 40.8 us).
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
        const long long slots = 4LL * nsm;
        auto cost = [&](int th, int tw) {
            const long long g = (long long)((m + th - 1) / th) * ((n + tw - 1) / tw) * batch;
            return ((g + slots - 1) / slots) * (long long)(th + 6) * (tw + 6);
        };
        const long long c32 = cost(32, 32), c64 = cost(32, 64), c28 = cost(28, 64);
        P->l1_wide = c64 < c32;
        P->l1_th = (c28 < c64 && c28 < c32) ? 28 : 0;
        if (const char* lw = getenv("CMG_L1_WIDE")) P->l1_wide = atoi(lw) != 0;
    }
    if (const char* rt = getenv("CMG_RP_TNT")) P->rp_tnt = atoi(rt);
    if (const char* lt = getenv("CMG_L1_TH")) P->l1_th = atoi(lt);
    if (const char* ll = getenv("CMG_L1_LOOP")) P->l1_loop = atoi(ll) != 0;
    if (const char* en = getenv("CMG_ENERGY_NT")) P->energy_nt = atoi(en) == 512 ? 512 : 256;
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
    NvtxRange nvtx("cmg_solve_device");
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
    NvtxRange nvtx("cmg_solve");
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
    P->hostP = sp;
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemcpyAsync(P->u, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->f, f_host, bytes, cudaMemcpyHostToDevice, P->stream));
    void* result = P->u;
    if (P->fused && layer <= 3 && ((P->fuse_mask >> (layer - 1)) & 1)) {
        if (P->dtype == CMG_F64)
            enqueue_fused_level<double>(P, layer, P->u, P->ubuf[2]);
        else
            enqueue_fused_level<float>(P, layer, P->u, P->ubuf[2]);
        result = P->ubuf[2];
    } else if (P->dtype == CMG_F64) {
        enqueue_fpads<double>(P);
        enqueue_fsums<double>(P);
        for (int c = 0; c < 4; ++c) enqueue_sweep<double>(P, layer, c);
    } else {
        enqueue_fpads<float>(P);
        enqueue_fsums<float>(P);
        for (int c = 0; c < 4; ++c) enqueue_sweep<float>(P, layer, c);
    }
    CK(cudaGetLastError());
    std::vector<ImgState> hs(P->B);
    CK(cudaMemcpyAsync(hs.data(), P->st, sizeof(ImgState) * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaMemcpyAsync(u_host, result, bytes, cudaMemcpyDeviceToHost, P->stream));
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
    P->hostP = sp;
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    CK(cudaMemcpyAsync(P->u, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->uprev, u_host, bytes, cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemcpyAsync(P->f, f_host, bytes, cudaMemcpyHostToDevice, P->stream));
    if (P->dtype == CMG_F64)
        enqueue_energy_ptrs<double>(P, P->u, P->uprev, false, P->eonly, 0, nullptr, 0, -1);
    else
        enqueue_energy_ptrs<float>(P, P->u, P->uprev, false, P->eonly, 0, nullptr, 0, -1);
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
    if (layer < 0 || layer > P->layers || color > 3 || reps < 1) return fail(CMG_EINVAL, "bad arguments");
    int rc = set_device(P);
    if (rc) return rc;
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    auto one = [&]() {
        if (layer == 0) {  // the energy + finalize kernel (energy-only output)
            if (P->dtype == CMG_F64)
                enqueue_energy_ptrs<double>(P, P->ubuf[0], P->ubuf[1], false, P->eonly, 0, nullptr, 0, -1);
            else
                enqueue_energy_ptrs<float>(P, P->ubuf[0], P->ubuf[1], false, P->eonly, 0, nullptr, 0, -1);
            return;
        }
        if (P->fused && layer <= 3 && ((P->fuse_mask >> (layer - 1)) & 1)) {  // production fused kernel
            if (P->dtype == CMG_F64)
                enqueue_fused_level<double>(P, layer, P->ubuf[0], P->ubuf[2]);
            else
                enqueue_fused_level<float>(P, layer, P->ubuf[0], P->ubuf[2]);
            return;
        }
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

static void* buffer_ptr(cmg_plan* P, int index) {
    if (index >= 0 && index <= 2) return P->ubuf[index];
    if (index == 3) return P->f;
    if (index == 5) return P->raw5;
    if (index == 4) {
        if (!P->ref) cudaMalloc(&P->ref, P->esz * (size_t)P->N * P->B);
        return P->ref;
    }
    return nullptr;
}

// NumPy pairwise summation tree (numpy/_core/src/umath/loops_utils.h.src):
// leaves of <= 128 elements in evaluation order, then the same recursion over
// the leaf sums
static void pairwise_leaves(long long off, long long n, std::vector<long long>& lo, std::vector<int>& ln) {
    if (n <= 128) {
        lo.push_back(off);
        ln.push_back((int)n);
        return;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    pairwise_leaves(off, n2, lo, ln);
    pairwise_leaves(off + n2, n - n2, lo, ln);
}
static double pairwise_combine(long long n, const double* leaf, size_t& next) {
    if (n <= 128) return leaf[next++];
    long long n2 = n / 2;
    n2 -= n2 % 8;
    const double l = pairwise_combine(n2, leaf, next);
    const double r = pairwise_combine(n - n2, leaf, next);
    return l + r;
}

// SSIM of batch image pairs already on the device (see cmg_metrics.cuh)
static int ssim_device(int batch, int m, int n, int dtype, const void* a, const void* b, const double* window,
                       double c1, double c2, double* out, cudaStream_t st) {
    const long long nout = (long long)(m - 10) * (n - 10);
    std::vector<long long> lo;
    std::vector<int> ln;
    pairwise_leaves(0, nout, lo, ln);
    const int nl = (int)lo.size();
    double *map = nullptr, *leaf = nullptr;
    long long* dlo = nullptr;
    int* dln = nullptr;
    auto cleanup = [&]() {
        cudaFree(map);
        cudaFree(leaf);
        cudaFree(dlo);
        cudaFree(dln);
    };
    cudaError_t e = cudaMalloc(&map, sizeof(double) * nout * batch);
    if (e == cudaSuccess) e = cudaMalloc(&leaf, sizeof(double) * nl * batch);
    if (e == cudaSuccess) e = cudaMalloc(&dlo, sizeof(long long) * nl);
    if (e == cudaSuccess) e = cudaMalloc(&dln, sizeof(int) * nl);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dlo, lo.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dln, ln.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        cleanup();
        return fail(CMG_ECUDA, cudaGetErrorString(e));
    }
    cmg::SsimArgs sa;
    for (int i = 0; i < 11; ++i) sa.w[i] = window[i];
    sa.c1 = c1;
    sa.c2 = c2;
    sa.m = m;
    sa.n = n;
    const dim3 g1((unsigned)((nout + 255) / 256), batch);
    if (dtype == CMG_F64)
        cmg::k_ssim_map<double><<<g1, 256, 0, st>>>((const double*)a, (const double*)b, map, sa);
    else
        cmg::k_ssim_map<float><<<g1, 256, 0, st>>>((const float*)a, (const float*)b, map, sa);
    cmg::k_pairwise_leaves<<<dim3((nl + 255) / 256, batch), 256, 0, st>>>(map, nout, dlo, dln, nl, leaf);
    std::vector<double> hl((size_t)nl * batch);
    e = cudaMemcpyAsync(hl.data(), leaf, sizeof(double) * nl * batch, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    cleanup();
    if (e != cudaSuccess) return fail(CMG_ECUDA, cudaGetErrorString(e));
    for (int bb = 0; bb < batch; ++bb) {
        size_t next = 0;
        out[bb] = pairwise_combine(nout, hl.data() + (size_t)bb * nl, next) / (double)nout;  // np.mean
    }
    return CMG_OK;
}

int cmg_ssim_batch(int batch, int m, int n, int dtype, const void* a_host, const void* b_host, const double* window,
                   double c1, double c2, double* out) {
    if (!a_host || !b_host || !window || !out) return fail(CMG_EINVAL, "NULL argument");
    if (batch < 1) return fail(CMG_EINVAL, "batch must be positive");
    if (dtype != CMG_F64 && dtype != CMG_F32) return fail(CMG_EINVAL, "dtype must be f64 or f32");
    if (m < 11 || n < 11) return fail(CMG_EINVAL, "image smaller than the 11x11 SSIM window");
    const size_t bytes = (size_t)(dtype == CMG_F64 ? 8 : 4) * m * n * batch;
    void *da = nullptr, *db = nullptr;
    cudaError_t e = cudaMalloc(&da, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&db, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(da, a_host, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(db, b_host, bytes, cudaMemcpyHostToDevice);
    int rc = (e == cudaSuccess) ? ssim_device(batch, m, n, dtype, da, db, window, c1, c2, out, 0)
                                : fail(CMG_ECUDA, cudaGetErrorString(e));
    cudaFree(da);
    cudaFree(db);
    return rc;
}

int cmg_plan_ssim(cmg_plan* P, int a_index, int b_index, const double* window, double c1, double c2, double* out) {
    if (!P || !window || !out) return fail(CMG_EINVAL, "NULL argument");
    int rc = set_device(P);
    if (rc) return rc;
    if (P->m < 11 || P->n < 11) return fail(CMG_EINVAL, "image smaller than the 11x11 SSIM window");
    if (a_index < 0 || a_index > 4 || b_index < 0 || b_index > 4) return fail(CMG_EINVAL, "buffer index must be 0..4");
    const void* a = buffer_ptr(P, a_index);
    const void* b = buffer_ptr(P, b_index);
    if (!a || !b) return fail(CMG_EINVAL, "buffer index must be 0..4");
    return ssim_device(P->B, P->m, P->n, P->dtype, a, b, window, c1, c2, out, P->stream);
}

int cmg_plan_buffer(cmg_plan* P, int index, void** dev_ptr) {
    if (!P || !dev_ptr) return fail(CMG_EINVAL, "NULL argument");
    int rc = set_device(P);
    if (rc) return rc;
    void* p = buffer_ptr(P, index);
    if (!p) return fail(CMG_EINVAL, "buffer index must be 0..4");
    *dev_ptr = p;
    return CMG_OK;
}

int cmg_buffer_upload(cmg_plan* P, int index, const void* host) {
    if (!P || !host) return fail(CMG_EINVAL, "NULL argument");
    if (index < 0 || index > 4) return fail(CMG_EINVAL, "buffer index must be 0..4");
    int rc = set_device(P);
    if (rc) return rc;
    void* p = buffer_ptr(P, index);
    if (!p) return fail(CMG_EINVAL, "buffer index must be 0..4");
    CK(cudaMemcpyAsync(p, host, P->esz * (size_t)P->N * P->B, cudaMemcpyHostToDevice, P->stream));
    if (index == 3) {  // f changed: refresh the padded f of general levels and the patch sums of f
        if (P->dtype == CMG_F64) {
            enqueue_fpads<double>(P);
            enqueue_fsums<double>(P);
        } else {
            enqueue_fpads<float>(P);
            enqueue_fsums<float>(P);
        }
    }
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

int cmg_buffer_download(cmg_plan* P, int index, void* host) {
    if (!P || !host) return fail(CMG_EINVAL, "NULL argument");
    if (index < 0 || index > 4) return fail(CMG_EINVAL, "buffer index must be 0..4");
    int rc = set_device(P);
    if (rc) return rc;
    void* p = buffer_ptr(P, index);
    if (!p) return fail(CMG_EINVAL, "buffer index must be 0..4");
    CK(cudaMemcpyAsync(host, p, P->esz * (size_t)P->N * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

int cmg_level_step(cmg_plan* P, int layer, int in_index, int out_index, double alpha, int inner_iters) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    if (layer < 1 || layer > P->layers) return fail(CMG_EINVAL, "layer outside the plan's hierarchy");
    if (in_index < 0 || in_index > 2 || out_index < 0 || out_index > 2 || in_index == out_index)
        return fail(CMG_EINVAL, "in/out must be distinct rotation buffers 0..2");
    int rc = check_cfg(alpha, 1.0, 1, inner_iters, 0);
    if (rc) return rc;
    rc = set_device(P);
    if (rc) return rc;
    SolveParams sp;
    fill_params(P, sp, alpha, 1.0, 1, inner_iters, 0, false, 1.0);
    P->hostP = sp;
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    enqueue_level(P, layer, in_index, out_index);
    CK(cudaGetLastError());
    std::vector<ImgState> hs(P->B);
    CK(cudaMemcpyAsync(hs.data(), P->st, sizeof(ImgState) * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    for (int b = 0; b < P->B; ++b)
        if (hs[b].bad) return fail(CMG_ENONFINITE, "corrections must be finite");
    return CMG_OK;
}

int cmg_energy_partials(cmg_plan* P, int u_index, int prev_index, int use_ref, int row_lo, int row_hi,
                        double* out) {
    if (!P || !out) return fail(CMG_EINVAL, "NULL argument");
    if (u_index < 0 || u_index > 2 || prev_index < 0 || prev_index > 2) return fail(CMG_EINVAL, "bad buffer index");
    if (row_lo < 0 || row_hi > P->m || row_lo > row_hi) return fail(CMG_EINVAL, "bad row range");
    int rc = set_device(P);
    if (rc) return rc;
    if (use_ref && !P->ref) return fail(CMG_EINVAL, "no reference uploaded (buffer 4)");
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    const long long lo = (long long)row_lo * P->n, hi = (long long)row_hi * P->n;
    if (P->dtype == CMG_F64)
        enqueue_energy_ptrs<double>(P, P->ubuf[u_index], P->ubuf[prev_index], use_ref != 0, nullptr, 0, P->raw5, lo, hi);
    else
        enqueue_energy_ptrs<float>(P, P->ubuf[u_index], P->ubuf[prev_index], use_ref != 0, nullptr, 0, P->raw5, lo, hi);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, P->raw5, sizeof(double) * NSUM * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

int cmg_l2_read_bandwidth(int device, long long bytes, int reps, double* gbs) {
    if (!gbs || bytes < (1 << 20) || reps < 1) return fail(CMG_EINVAL, "bad arguments");
    CK(cudaSetDevice(device));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const long long n16 = bytes / 16;
    uint4* buf = nullptr;
    unsigned* sink = nullptr;
    CK(cudaMalloc(&buf, n16 * 16));
    if (cudaMalloc(&sink, sizeof(unsigned) * 1024 * 1024) != cudaSuccess) {
        cudaFree(buf);
        return fail(CMG_ECUDA, "cudaMalloc");
    }
    cudaStream_t st;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemsetAsync(buf, 1, n16 * 16, st);
    const int grid = nsm * 8;
    k_l2_read<<<grid, 256, 0, st>>>(buf, n16, 1, sink);  // warm: the buffer is L2-resident afterwards
    cudaEventRecord(e0, st);
    k_l2_read<<<grid, 256, 0, st>>>(buf, n16, reps, sink);
    cudaEventRecord(e1, st);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    cudaFree(buf);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(CMG_ECUDA, cudaGetErrorString(e));
    *gbs = (double)n16 * 16.0 * reps / (ms * 1e-3) / 1e9;
    return CMG_OK;
}

int cmg_fp64_probe(int device, double* dfma_per_clk_per_sm, double* dep_latency_cycles, double* tflops) {
    if (!dfma_per_clk_per_sm || !dep_latency_cycles || !tflops) return fail(CMG_EINVAL, "NULL argument");
    CK(cudaSetDevice(device));
    int nsm = 0, khz = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device));
    double* out = nullptr;
    long long* cyc = nullptr;
    CK(cudaMalloc(&out, sizeof(double) * (size_t)nsm * 4 * 1024));
    if (cudaMalloc(&cyc, sizeof(long long)) != cudaSuccess) {
        cudaFree(out);
        return fail(CMG_ECUDA, "cudaMalloc");
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    // latency: one warp, one chain; (cycles between the clock reads) / iters
    k_fp64_chain<1><<<1, 32>>>(out, iters, 0.999, 1e-9, cyc);
    k_fp64_chain<1><<<1, 32>>>(out, iters, 0.999, 1e-9, cyc);
    long long hc = 0;
    cudaError_t e = cudaMemcpy(&hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    // throughput: 4 CTAs of 1024 threads per SM (all 64 warps), 8 chains per thread
    k_fp64_chain<8><<<nsm * 4, 1024>>>(out, 64, 0.999, 1e-9, nullptr);
    cudaEventRecord(e0);
    k_fp64_chain<8><<<nsm * 4, 1024>>>(out, iters, 0.999, 1e-9, nullptr);
    cudaEventRecord(e1);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaFree(cyc);
    if (e != cudaSuccess) return fail(CMG_ECUDA, cudaGetErrorString(e));
    const double dfma = (double)nsm * 4 * 1024 * 8.0 * iters;  // thread-level DFMAs
    *dep_latency_cycles = (double)hc / iters;
    *tflops = 2.0 * dfma / (ms * 1e-3) / 1e12;
    *dfma_per_clk_per_sm = dfma / (ms * 1e-3) / ((double)khz * 1e3) / nsm;
    return CMG_OK;
}

int cmg_plan_stream(cmg_plan* P, void** stream) {
    if (!P || !stream) return fail(CMG_EINVAL, "NULL argument");
    *stream = (void*)P->stream;
    return CMG_OK;
}

int cmg_strip_begin(cmg_plan* P, double alpha, int inner_iters) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    int rc = check_cfg(alpha, 1.0, 1, inner_iters, 0);
    if (rc) return rc;
    rc = set_device(P);
    if (rc) return rc;
    SolveParams sp;
    fill_params(P, sp, alpha, 1.0, 1, inner_iters, 0, false, 1.0);
    P->hostP = sp;
    CK(cudaMemcpyAsync(P->P, &sp, sizeof(sp), cudaMemcpyHostToDevice, P->stream));
    CK(cudaMemsetAsync(P->st, 0, sizeof(ImgState) * P->B, P->stream));
    // the host struct must outlive the async copy: make this call synchronous once
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

int cmg_level_step_async(cmg_plan* P, int layer, int in_index, int out_index) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    if (layer < 1 || layer > P->layers) return fail(CMG_EINVAL, "layer outside the plan's hierarchy");
    if (in_index < 0 || in_index > 2 || out_index < 0 || out_index > 2 || in_index == out_index)
        return fail(CMG_EINVAL, "in/out must be distinct rotation buffers 0..2");
    int rc = set_device(P);
    if (rc) return rc;
    enqueue_level(P, layer, in_index, out_index);
    CK(cudaGetLastError());
    return CMG_OK;
}

int cmg_strip_partials_async(cmg_plan* P, int u_index, int prev_index, int use_ref, int row_lo, int row_hi) {
    if (!P) return fail(CMG_EINVAL, "plan is NULL");
    if (u_index < 0 || u_index > 2 || prev_index < 0 || prev_index > 2) return fail(CMG_EINVAL, "bad buffer index");
    if (row_lo < 0 || row_hi > P->m || row_lo > row_hi) return fail(CMG_EINVAL, "bad row range");
    if (use_ref && !P->ref) return fail(CMG_EINVAL, "no reference uploaded (buffer 4)");
    int rc = set_device(P);
    if (rc) return rc;
    const long long lo = (long long)row_lo * P->n, hi = (long long)row_hi * P->n;
    if (P->dtype == CMG_F64)
        enqueue_energy_ptrs<double>(P, P->ubuf[u_index], P->ubuf[prev_index], use_ref != 0, nullptr, 0, P->raw5, lo, hi);
    else
        enqueue_energy_ptrs<float>(P, P->ubuf[u_index], P->ubuf[prev_index], use_ref != 0, nullptr, 0, P->raw5, lo, hi);
    k_strip_flags<<<(P->B + 127) / 128, 128, 0, P->stream>>>(P->st, P->raw5, P->B);
    CK(cudaGetLastError());
    return CMG_OK;
}

int cmg_strip_read(cmg_plan* P, double* out) {
    if (!P || !out) return fail(CMG_EINVAL, "NULL argument");
    int rc = set_device(P);
    if (rc) return rc;
    CK(cudaMemcpyAsync(out, P->raw5, sizeof(double) * (NSUM + 1) * P->B, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    return CMG_OK;
}

}  // extern "C"

struct cmg_mplan {
    int m = 0, n = 0, B = 0, esz = 8;
    std::vector<cmg_plan*> plans;
    std::vector<int> off, cnt;
};

extern "C" {

int cmg_mplan_destroy(cmg_mplan* M) {
    if (!M) return CMG_OK;
    for (cmg_plan* p : M->plans) cmg_plan_destroy(p);
    delete M;
    return CMG_OK;
}

int cmg_mplan_create(cmg_mplan** out, int m, int n, int batch, int layers, int mode, int dtype, int precision,
                     const int* device_ids, int n_devices) {
    if (!out) return fail(CMG_EINVAL, "out is NULL");
    *out = nullptr;
    if (!device_ids || n_devices < 1) return fail(CMG_EINVAL, "need at least one device id");
    if (batch < n_devices) return fail(CMG_EINVAL, "batch must be at least the number of devices");
    cmg_mplan* M = new cmg_mplan();
    M->m = m;
    M->n = n;
    M->B = batch;
    M->esz = dtype == CMG_F64 ? 8 : 4;
    int o = 0;
    for (int d = 0; d < n_devices; ++d) {
        const int c = batch / n_devices + (d < batch % n_devices ? 1 : 0);
        cmg_plan* p = nullptr;
        const int rc = cmg_plan_create(&p, m, n, c, layers, mode, dtype, precision, device_ids[d]);
        if (rc != CMG_OK) {
            cmg_mplan_destroy(M);
            return rc;
        }
        M->plans.push_back(p);
        M->off.push_back(o);
        M->cnt.push_back(c);
        o += c;
    }
    *out = M;
    return CMG_OK;
}

int cmg_mplan_solve(cmg_mplan* M, const void* f_host, const void* ref_host, void* u_host_out, double alpha,
                    double epsilon, int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak,
                    double* energy, double* rel_energy, double* rel_u, double* psnr, double* seconds, int* iterations,
                    int* status) {
    if (!M) return fail(CMG_EINVAL, "plan is NULL");
    if (!f_host) return fail(CMG_EINVAL, "f is NULL");
    const int nd = (int)M->plans.size();
    const size_t img = (size_t)M->m * M->n * M->esz;
    const size_t cap = (size_t)max_outer + 1;
    std::vector<int> rcs(nd, CMG_OK);
    std::vector<std::string> errs(nd);
    std::vector<int> st(M->B, CMG_OK);
    auto shard = [&](int d) {
        const size_t o = (size_t)M->off[d];
        auto tr = [&](double* a) { return a ? a + o * cap : nullptr; };
        rcs[d] = cmg_solve(M->plans[d], (const char*)f_host + o * img, ref_host ? (const char*)ref_host + o * img : nullptr,
                           u_host_out ? (char*)u_host_out + o * img : nullptr, alpha, epsilon, max_outer, inner_iters,
                           stop_rule, full_vcycle, peak, tr(energy), tr(rel_energy), tr(rel_u), tr(psnr), tr(seconds),
                           iterations ? iterations + o : nullptr, st.data() + o);
        if (rcs[d] == CMG_EINVAL || rcs[d] == CMG_ECUDA) errs[d] = g_err;
    };
    std::vector<std::thread> th;
    for (int d = 1; d < nd; ++d) th.emplace_back(shard, d);
    shard(0);
    for (auto& t : th) t.join();
    for (int d = 0; d < nd; ++d)
        if (rcs[d] == CMG_EINVAL || rcs[d] == CMG_ECUDA) return fail(rcs[d], errs[d]);
    if (status)
        for (int b = 0; b < M->B; ++b) status[b] = st[b];
    for (int b = 0; b < M->B; ++b)
        if (st[b] != CMG_OK) {
            if (st[b] == CMG_DIVERGED) g_err = "objective became non-finite";
            if (st[b] == CMG_ENONFINITE) g_err = "corrections must be finite";
            return st[b];
        }
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
