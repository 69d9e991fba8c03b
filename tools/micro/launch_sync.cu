// Microbenchmarks: dependent-kernel launch cost inside a CUDA graph, and
// cooperative grid.sync() cost, on the local GPU.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_empty(int* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++; }
__global__ void k_work(double* a, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = a[i] * 1.0000001 + 1e-9;
}
__global__ void k_sync(int iters, int* x) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) atomicAdd(x + (blockIdx.x & 7), 1);
        g.sync();
    }
}

int main() {
    int* x; double* a;
    cudaMalloc(&x, 64); cudaMalloc(&a, sizeof(double) * (1 << 20));
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int grid : {1, 148, 1184, 4096}) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 100; ++i) k_empty<<<grid, 256, 0, s>>>(x);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("graph empty kernel grid=%d: %.3f us per kernel\n", grid, ms * 1000 / 1000);
    }
    {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 100; ++i) k_work<<<4096, 256, 0, s>>>(a, 1 << 20);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("graph 1M-double axpy kernel: %.3f us per kernel\n", ms * 1000 / 1000);
    }
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {1, 2, 4, 8}) {
        int iters = 1000; int grid = nsm * per;
        void* args[] = {&iters, &x};
        cudaLaunchCooperativeKernel((void*)k_sync, grid, 256, args, 0, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        cudaLaunchCooperativeKernel((void*)k_sync, grid, 256, args, 0, s);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("grid.sync grid=%d: %.3f us per sync (%s)\n", grid, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
