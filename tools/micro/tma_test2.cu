// TMA 3-D load variants (debugging): argv[1] selects the variant.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ CUtensorMap g_tm;
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int box, int x0, int y0) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* s = reinterpret_cast<float*>(sm + 1024);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm);
    const CUtensorMap* mp = (V & 1) ? &g_tm : &tm;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(mp) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(box * box * 4) : "memory");
        if (V & 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(s)), "l"(mp), "r"(x0), "r"(y0), "r"(smem_u32(bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(smem_u32(s)), "l"(mp), "r"(x0), "r"(y0), "r"(0), "r"(smem_u32(bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < box * box; i += blockDim.x) out[i] = s[i];
}
typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    int V = atoi(argv[1]);
    int x0 = argc > 2 ? atoi(argv[2]) : -3, y0 = argc > 3 ? atoi(argv[3]) : -5;
    int m = 512, n = 512; int box = argc > 4 ? atoi(argv[4]) : 36;
    std::vector<float> h(m * n);
    for (int i = 0; i < m * n; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, m * n * 4); cudaMalloc(&o, box * box * 4);
    cudaMemcpy(d, h.data(), m * n * 4, cudaMemcpyHostToDevice);
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm;
    int rank = (V & 2) ? 2 : 3;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, 1}, str[2] = {(cuuint64_t)n * 4, (cuuint64_t)m * n * 4};
    cuuint32_t bx[3] = {(cuuint32_t)box, (cuuint32_t)box, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Fn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpyToSymbol(g_tm, &tm, sizeof(tm));
    size_t smem = 1024 + box * box * 4;
    auto kk = V == 0 ? k<0> : V == 1 ? k<1> : V == 2 ? k<2> : k<3>;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kk<<<1, 128, smem>>>(tm, o, box, x0, y0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(box * box);
    cudaMemcpy(ho.data(), o, box * box * 4, cudaMemcpyDeviceToHost);
    int yy = 6, xx = 4; (void)0;
    printf("V=%d x0=%d y0=%d encode=%d: %s  s[6][4]=%g (expect %d)\n", V, x0, y0, (int)r, cudaGetErrorString(e), ho[yy*box+xx], (y0+yy)*512 + (x0+xx));
    return e != cudaSuccess;
}
