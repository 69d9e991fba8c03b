// double instantiation of the launch sequences
#include "cmg_launch.cuh"
CMG_INSTANTIATE(double)

// Self test of the branch-free correctly rounded sqrt / div (cmg_l1loop.cuh)
// against __dsqrt_rn / __ddiv_rn on n host operand pairs: out[0] / out[1] =
// in-range sqrt(a) / a/b results that differ from the library (must be 0),
// out[2] / out[3] = operands the range tests send to the library path.
extern "C" int cmg_selftest_exact(int device, const double* a_host, const double* b_host, long long n,
                                  unsigned long long* out) {
    if (!a_host || !b_host || !out || n < 1) return CMG_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return CMG_ECUDA;
    double *a = nullptr, *b = nullptr;
    unsigned long long* o = nullptr;
    cudaError_t e = cudaMalloc(&a, n * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&b, n * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&o, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpy(a, a_host, n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(b, b_host, n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(o, 0, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) {
        cmg::k_selftest_exact<<<592, 256>>>(a, b, n, o);
        e = cudaDeviceSynchronize();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, o, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(a);
    cudaFree(b);
    cudaFree(o);
    return e == cudaSuccess ? CMG_OK : CMG_ECUDA;
}
