// TMA: two boxes (u and f) into one mbarrier, like k_coarse_tile.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
template <typename T>
__global__ void k(const __grid_constant__ CUtensorMap tu, const __grid_constant__ CUtensorMap tf, T* out, int box, int x0, int y0, int cells_al) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* b128 = sm + ((128 - (smem_u32(sm) & 127)) & 127);
    T* su = reinterpret_cast<T*>(b128);
    T* sf = su + cells_al;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sf + cells_al);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(2 * box * box * (int)sizeof(T)) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(smem_u32(su)), "l"(&tu), "r"(x0), "r"(y0), "r"(0), "r"(smem_u32(bar)) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(smem_u32(sf)), "l"(&tf), "r"(x0), "r"(y0), "r"(0), "r"(smem_u32(bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < box * box; i += blockDim.x) out[i] = su[i] + sf[i];
}
typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
template <typename T>
int run(int box, int x0, int y0) {
    int m = 1024, n = 1024;
    std::vector<T> h(m * n);
    for (int i = 0; i < m * n; ++i) h[i] = i;
    T *du, *df, *o;
    cudaMalloc(&du, m * n * sizeof(T)); cudaMalloc(&df, m * n * sizeof(T)); cudaMalloc(&o, box * box * sizeof(T));
    cudaMemcpy(du, h.data(), m * n * sizeof(T), cudaMemcpyHostToDevice);
    cudaMemcpy(df, h.data(), m * n * sizeof(T), cudaMemcpyHostToDevice);
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tu, tf;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, 1}, str[2] = {(cuuint64_t)n * sizeof(T), (cuuint64_t)m * n * sizeof(T)};
    cuuint32_t bx[3] = {(cuuint32_t)box, (cuuint32_t)box, 1}, es[3] = {1, 1, 1};
    CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r1 = ((Fn)p)(&tu, dt, 3, du, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = ((Fn)p)(&tf, dt, 3, df, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int cells = box * box;
    int cells_al = (cells * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
    size_t smem = 128 + 2 * sizeof(T) * cells_al + 16;
    cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<T><<<1, 256, smem>>>(tu, tf, o, box, x0, y0, cells_al);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<T> ho(box * box);
    cudaMemcpy(ho.data(), o, box * box * sizeof(T), cudaMemcpyDeviceToHost);
    printf("esz=%d box=%d x0=%d y0=%d enc=%d,%d smem=%zu: %s  v=%g expect %g\n", (int)sizeof(T), box, x0, y0, (int)r1, (int)r2, smem, cudaGetErrorString(e), (double)ho[6 * box + 4], 2.0 * ((y0 + 6) * 1024 + x0 + 4));
    return e != cudaSuccess;
}
int main(int argc, char** argv) {
    int es = atoi(argv[1]), box = atoi(argv[2]), x0 = atoi(argv[3]), y0 = atoi(argv[4]);
    return es == 8 ? run<double>(box, x0, y0) : run<float>(box, x0, y0);
}
