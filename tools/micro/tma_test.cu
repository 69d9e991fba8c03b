// Minimal TMA 3-D load test (debugging the coarse-tile staging path).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int box, int x0, int y0) {
    extern __shared__ __align__(128) unsigned char sm[];
    float* s = reinterpret_cast<float*>(sm);
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        if (V == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(box * box * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(smem_u32(s)), "l"(&tm), "r"(x0), "r"(y0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < box * box; i += blockDim.x) out[i] = s[i];
}
typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    int m = 64, n = 64, box = 36;
    std::vector<float> h(m * n);
    for (int i = 0; i < m * n; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, m * n * 4); cudaMalloc(&o, box * box * 4);
    cudaMemcpy(d, h.data(), m * n * 4, cudaMemcpyHostToDevice);
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, 1}, str[2] = {(cuuint64_t)n * 4, (cuuint64_t)m * n * 4};
    cuuint32_t bx[3] = {(cuuint32_t)box, (cuuint32_t)box, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Fn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int v = 1; v >= 0; --v) {
        if (v == 1) k<1><<<1, 128, box * box * 4>>>(tm, o, box, -3, -5);
        else k<0><<<1, 128, box * box * 4>>>(tm, o, box, -3, -5);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> ho(box * box);
        cudaMemcpy(ho.data(), o, box * box * 4, cudaMemcpyDeviceToHost);
        printf("variant %d: %s  s[0]=%g s[5*36+3]=%g (expect 0 and 0) s[6*36+4]=%g (expect %d)\n", v, cudaGetErrorString(e), ho[0], ho[5*36+3], ho[6*36+4], 1*64+1);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
