// cmg_recon.cu -- device operators of the curvature-regularised
// reconstruction (reference curvemg.reconstruction, reconstruction.py):
//
//   parallel-beam Radon transform (reconstruction.py:123-183): pixel-driven
//     linear splat onto the two nearest detector bins.  The forward is a
//     deterministic GATHER: per (angle, bin) the pixels whose lower bin is
//     this bin (or the one below) are summed in increasing pixel order --
//     exactly np.bincount's accumulation order, so sinograms are bit-identical
//     to the reference's.  The adjoint gathers per pixel over the angles in
//     order (`out += row[i0]*(1-w) + row[i0+1]*w`), also bit-identical.
//   per-colour pieces of the multigrid step (reconstruction.py:389-431):
//     mean plane distance d at every patch centre of one colour (the
//     distance_fields + mean of the denoiser, exact operation order), the
//     piecewise-constant prolongation u + P c, and patch sums of an image.
//   the level-1 mean-curvature mass (tangent.curvature_field, closed form).
//
// fp64 only (the reference computes in float64).  Vector algebra (CG) and the
// masked FFT run on the same CUDA stream through PyTorch (cuBLAS / cuFFT).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/cmg.h"
#include "cmg_kernels.cuh"

using namespace cmg;

namespace cmg {
int set_error(int code, const char* msg);
}

struct cmg_radon {
    int m = 0, n = 0, na = 0, nb = 0, device = 0;
    double ps = 0.0;
    int* i0 = nullptr;      // [na][m*n] lower detector bin of each pixel
    double* w = nullptr;    // [na][m*n] weight of the upper bin
    int* off = nullptr;     // [na][nb+1] CSR: pixels whose lower bin is k
    int* idx = nullptr;     // [na][m*n] pixel ids, ascending within a bin
};

namespace {

// sino[a][k] = sum_{i0_p == k} x_p ps (1 - w_p)  +  sum_{i0_p == k-1} x_p ps w_p
__global__ void k_radon_fwd(const double* __restrict__ x, double* __restrict__ sino, const int* __restrict__ off,
                            const int* __restrict__ idx, const double* __restrict__ w, int N, int nb, double ps) {
    const int a = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nb) return;
    const int* o = off + (long long)a * (nb + 1);
    const int* id = idx + (long long)a * N;
    const double* wa = w + (long long)a * N;
    double s1 = 0.0, s2 = 0.0;
    for (int t = o[k]; t < o[k + 1]; ++t) {
        const int p = id[t];
        s1 = __dadd_rn(s1, __dmul_rn(__dmul_rn(x[p], ps), __dsub_rn(1.0, wa[p])));
    }
    if (k >= 1)
        for (int t = o[k - 1]; t < o[k]; ++t) {
            const int p = id[t];
            s2 = __dadd_rn(s2, __dmul_rn(__dmul_rn(x[p], ps), wa[p]));
        }
    sino[(long long)a * nb + k] = __dadd_rn(s1, s2);
}

// out_p = ps * sum_a (y[a][i0] (1 - w) + y[a][i0 + 1] w), angles in order
__global__ void k_radon_adj(const double* __restrict__ y, double* __restrict__ out, const int* __restrict__ i0,
                            const double* __restrict__ w, int N, int na, int nb, double ps) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double acc = 0.0;
    for (int a = 0; a < na; ++a) {
        const long long e = (long long)a * N + p;
        const int b = i0[e];
        const double wv = w[e];
        const double* row = y + (long long)a * nb;
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(row[b], __dsub_rn(1.0, wv)), __dmul_rn(row[b + 1], wv)));
    }
    out[p] = __dmul_rn(acc, ps);
}

// mean perpendicular plane distance at the centre of every patch of colour
// (p, q) of level `layer` (tangent.distance_fields + d.mean(axis=0), the
// denoiser's operation order; a single-patch class sums pairwise)
__global__ void k_recon_chalf(const double* __restrict__ u, int m, int n, int layer, int p, int q, int hc, int wc,
                              double* __restrict__ d) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hc * wc) return;
    const int S = (1 << layer) - 1, R = 1 << (layer - 1), npl = 1 << (layer + 2);
    const int a = e / wc, bq = e % wc;
    const int ci = (2 * a + p) * S + R - 1, cc = (2 * bq + q) * S + R - 1;
    const Reflect<double> U{u, m, n};
    const double uo = U(ci, cc);
    double sum;
    if (hc * wc == 1) {
        sum = pairwise_any<double>(npl, [&](int l) {
            double v;
            plane_exact_rt<double>(U, ci, cc, uo, PlaneRT::getg(l), &v, nullptr);
            return v;
        });
    } else {
        plane_exact_rt<double>(U, ci, cc, uo, PlaneRT::getg(0), &sum, nullptr);
        for (int l = 1; l < npl; ++l) {
            double v;
            plane_exact_rt<double>(U, ci, cc, uo, PlaneRT::getg(l), &v, nullptr);
            sum = __dadd_rn(sum, v);
        }
    }
    d[e] = __ddiv_rn(sum, (double)npl);
}

// u + prolong(c): every pixel gets + c of its patch if the patch has colour
// (p, q), else + 0.0 (as the reference's dense `u + cfull` expansion)
__global__ void k_recon_prolong(double* __restrict__ u, const double* __restrict__ c, int m, int n, int S, int p,
                                int q, int wc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)m * n) return;
    const int i = (int)(e / n), k = (int)(e % n);
    const int pi = i / S, pk = k / S;
    double add = 0.0;
    if ((pi & 1) == p && (pk & 1) == q) add = c[(long long)(pi >> 1) * wc + (pk >> 1)];
    u[e] = __dadd_rn(u[e], add);
}

// per-patch sums (zero padding beyond the image) for the patches of colour (p, q)
__global__ void k_recon_block_sums(const double* __restrict__ img, int m, int n, int S, int p, int q, int hc, int wc,
                                   double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hc * wc) return;
    const int r0 = (2 * (e / wc) + p) * S, c0 = (2 * (e % wc) + q) * S;
    double s = 0.0;
    for (int i = r0; i < r0 + S && i < m; ++i)
        for (int k = c0; k < c0 + S && k < n; ++k) s = __dadd_rn(s, img[(long long)i * n + k]);
    out[e] = s;
}

// level-1 mean-curvature mass: per-block partial sums of |0.5 (kmin + kmax)|
__global__ void k_recon_curv(const double* __restrict__ u, int m, int n, double* __restrict__ partial) {
    __shared__ double sh[256];
    const Reflect<double> U{u, m, n};
    double acc = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)m * n;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), k = (int)(e % n);
        acc += curv_term<double>(U(i, k), U(i, k + 1), U(i, k - 1), U(i - 1, k), U(i + 1, k), U(i - 1, k + 1),
                                 U(i + 1, k - 1), U(i - 1, k - 1), U(i + 1, k + 1), MODE_MEAN);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

inline bool single_chunk(int len) { return len >= 2; }

}  // namespace

#define RCK(x)                                                                            \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) return cmg::set_error(CMG_ECUDA, cudaGetErrorString(e_)); \
    } while (0)

extern "C" {

int cmg_radon_destroy(cmg_radon* R) {
    if (!R) return CMG_OK;
    cudaSetDevice(R->device);
    cudaFree(R->i0);
    cudaFree(R->w);
    cudaFree(R->off);
    cudaFree(R->idx);
    delete R;
    return CMG_OK;
}

int cmg_radon_create(cmg_radon** out, int m, int n, int n_angles, int detector_count, double pixel_size,
                     const int* i0_host, const double* w_host, int device) {
    if (!out || !i0_host || !w_host) return cmg::set_error(CMG_EINVAL, "NULL argument");
    *out = nullptr;
    if (m < 1 || n < 1 || n_angles < 1 || detector_count < 2 || !(pixel_size > 0))
        return cmg::set_error(CMG_EINVAL, "bad Radon geometry");
    const long long N = (long long)m * n;
    if (N * n_angles >= (1LL << 31)) return cmg::set_error(CMG_EINVAL, "Radon operator too large");
    // CSR of pixels per (angle, lower bin), ascending pixel order (np.bincount order)
    std::vector<int> off((size_t)n_angles * (detector_count + 1), 0), idx((size_t)n_angles * N);
    for (int a = 0; a < n_angles; ++a) {
        const int* ia = i0_host + (size_t)a * N;
        int* oa = off.data() + (size_t)a * (detector_count + 1);
        for (long long p = 0; p < N; ++p) {
            if (ia[p] < 0 || ia[p] + 1 >= detector_count)
                return cmg::set_error(CMG_EINVAL, "detector does not cover the image; enlarge detector_count");
            oa[ia[p] + 1]++;
        }
        for (int k = 0; k < detector_count; ++k) oa[k + 1] += oa[k];
        std::vector<int> fill(oa, oa + detector_count);
        int* xa = idx.data() + (size_t)a * N;
        for (long long p = 0; p < N; ++p) xa[fill[ia[p]]++] = (int)p;
    }
    cmg_radon* R = new cmg_radon();
    R->m = m;
    R->n = n;
    R->na = n_angles;
    R->nb = detector_count;
    R->ps = pixel_size;
    R->device = device;
    auto bail = [&](cudaError_t e) {
        cmg_radon_destroy(R);
        return cmg::set_error(CMG_ECUDA, cudaGetErrorString(e));
    };
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&R->i0, sizeof(int) * N * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&R->w, sizeof(double) * N * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&R->off, sizeof(int) * off.size());
    if (e == cudaSuccess) e = cudaMalloc(&R->idx, sizeof(int) * idx.size());
    if (e == cudaSuccess) e = cudaMemcpy(R->i0, i0_host, sizeof(int) * N * n_angles, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(R->w, w_host, sizeof(double) * N * n_angles, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(R->off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(R->idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(e);
    *out = R;
    return CMG_OK;
}

int cmg_radon_forward(cmg_radon* R, const double* x_dev, double* sino_dev, void* stream) {
    if (!R || !x_dev || !sino_dev) return cmg::set_error(CMG_EINVAL, "NULL argument");
    RCK(cudaSetDevice(R->device));
    const dim3 g((R->nb + 127) / 128, R->na);
    k_radon_fwd<<<g, 128, 0, (cudaStream_t)stream>>>(x_dev, sino_dev, R->off, R->idx, R->w, R->m * R->n, R->nb,
                                                      R->ps);
    RCK(cudaGetLastError());
    return CMG_OK;
}

int cmg_radon_adjoint(cmg_radon* R, const double* y_dev, double* x_dev, void* stream) {
    if (!R || !y_dev || !x_dev) return cmg::set_error(CMG_EINVAL, "NULL argument");
    RCK(cudaSetDevice(R->device));
    const int N = R->m * R->n;
    k_radon_adj<<<(N + 255) / 256, 256, 0, (cudaStream_t)stream>>>(y_dev, x_dev, R->i0, R->w, N, R->na, R->nb,
                                                                    R->ps);
    RCK(cudaGetLastError());
    return CMG_OK;
}

int cmg_recon_chalf(const double* u_dev, int m, int n, int layer, int p, int q, double* d_dev, void* stream) {
    if (!u_dev || !d_dev) return cmg::set_error(CMG_EINVAL, "NULL argument");
    if (layer < 1 || layer > 6 || p < 0 || p > 1 || q < 0 || q > 1) return cmg::set_error(CMG_EINVAL, "bad level/colour");
    const int S = (1 << layer) - 1;
    const int mj = (m + S - 1) / S, nj = (n + S - 1) / S;
    const int hc = (mj - p + 1) / 2, wc = (nj - q + 1) / 2;
    // single-chunk odd reflection only (images of at least 2 x 2 and a padding
    // of at most len - 1 on every side); smaller images need numpy's iterated pad
    if (!single_chunk(m) || !single_chunk(n) || 1 + mj * S - m > m - 1 || 1 + nj * S - n > n - 1)
        return cmg::set_error(CMG_EINVAL, "image too small for this level on the GPU reconstruction path");
    if (hc <= 0 || wc <= 0) return CMG_OK;
    k_recon_chalf<<<(hc * wc + 127) / 128, 128, 0, (cudaStream_t)stream>>>(u_dev, m, n, layer, p, q, hc, wc, d_dev);
    RCK(cudaGetLastError());
    return CMG_OK;
}

int cmg_recon_prolong(double* u_dev, const double* c_dev, int m, int n, int layer, int p, int q, void* stream) {
    if (!u_dev || !c_dev) return cmg::set_error(CMG_EINVAL, "NULL argument");
    const int S = (1 << layer) - 1;
    const int nj = (n + S - 1) / S;
    const int wc = (nj - q + 1) / 2;
    const long long N = (long long)m * n;
    k_recon_prolong<<<(unsigned)((N + 255) / 256), 256, 0, (cudaStream_t)stream>>>(u_dev, c_dev, m, n, S, p, q, wc);
    RCK(cudaGetLastError());
    return CMG_OK;
}

int cmg_recon_block_sums(const double* img_dev, int m, int n, int layer, int p, int q, double* out_dev, void* stream) {
    if (!img_dev || !out_dev) return cmg::set_error(CMG_EINVAL, "NULL argument");
    const int S = (1 << layer) - 1;
    const int mj = (m + S - 1) / S, nj = (n + S - 1) / S;
    const int hc = (mj - p + 1) / 2, wc = (nj - q + 1) / 2;
    if (hc <= 0 || wc <= 0) return CMG_OK;
    k_recon_block_sums<<<(hc * wc + 127) / 128, 128, 0, (cudaStream_t)stream>>>(img_dev, m, n, S, p, q, hc, wc,
                                                                               out_dev);
    RCK(cudaGetLastError());
    return CMG_OK;
}

int cmg_recon_curvature_partials(const double* u_dev, int m, int n, double* partial_dev, int nblocks, void* stream) {
    if (!u_dev || !partial_dev || nblocks < 1) return cmg::set_error(CMG_EINVAL, "bad arguments");
    if (m < 2 || n < 2) return cmg::set_error(CMG_EINVAL, "image too small");
    k_recon_curv<<<nblocks, 256, 0, (cudaStream_t)stream>>>(u_dev, m, n, partial_dev);
    RCK(cudaGetLastError());
    return CMG_OK;
}

}  // extern "C"
