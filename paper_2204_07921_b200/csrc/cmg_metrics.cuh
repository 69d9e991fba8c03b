// cmg_metrics.cuh -- on-device image metrics of the denoising trace
// (SURVEY 8(f) rank 1): SSIM with the reference's operation order, so the
// result is bit-identical to curvemg.image.ssim (image.py:152-192).
//
//  * k_ssim_map: one thread per valid 11x11 window.  The separable filter of
//    _filter_valid (image.py:163-167) is restated term by term: rows first
//    (Python sum from 0: 0 + w0 a0 + w1 a1 + ...), then columns, for x, y,
//    x*x, y*y and x*y (each product rounded first, as NumPy evaluates it);
//    then var / cov / num / den / num/den in the reference's association
//    order, every operation separately rounded.
//  * k_pairwise_leaves: np.mean's pairwise sum (NumPy pairwise_sum, blocks of
//    <= 128 with eight accumulators) evaluated leaf by leaf; the host combines
//    the leaf sums along the same recursion (cmg.cu), then divides by N.
#pragma once

#include "cmg_device.cuh"

namespace cmg {

struct SsimArgs {
    double w[11];  // _gaussian_window(11, 1.5), computed by the caller exactly as the reference
    double c1, c2;  // (K1 peak)^2, (K2 peak)^2
    int m, n;       // image shape; the map is (m-10) x (n-10)
};

template <typename T>
__global__ void __launch_bounds__(256) k_ssim_map(const T* __restrict__ a, const T* __restrict__ b, double* map,
                                                  SsimArgs s) {
    pdl_sync();
    using O = X<double>;
    const int img = blockIdx.y;
    const int mo = s.m - 10, no = s.n - 10;
    const long long nout = (long long)mo * no;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nout) return;
    const int r = (int)(e / no), c = (int)(e % no);
    const T* x = a + (long long)img * s.m * s.n;
    const T* y = b + (long long)img * s.m * s.n;
    double fx = 0.0, fy = 0.0, fxx = 0.0, fyy = 0.0, fxy = 0.0;  // column pass accumulators
    for (int j = 0; j < 11; ++j) {
        double rx = 0.0, ry = 0.0, rxx = 0.0, ryy = 0.0, rxy = 0.0;  // row pass at column c+j
        for (int i = 0; i < 11; ++i) {
            const long long g = (long long)(r + i) * s.n + (c + j);
            const double xv = (double)x[g], yv = (double)y[g];
            const double wi = s.w[i];
            rx = O::add(rx, O::mul(wi, xv));
            ry = O::add(ry, O::mul(wi, yv));
            rxx = O::add(rxx, O::mul(wi, O::mul(xv, xv)));
            ryy = O::add(ryy, O::mul(wi, O::mul(yv, yv)));
            rxy = O::add(rxy, O::mul(wi, O::mul(xv, yv)));
        }
        const double wj = s.w[j];
        fx = O::add(fx, O::mul(wj, rx));
        fy = O::add(fy, O::mul(wj, ry));
        fxx = O::add(fxx, O::mul(wj, rxx));
        fyy = O::add(fyy, O::mul(wj, ryy));
        fxy = O::add(fxy, O::mul(wj, rxy));
    }
    const double var_x = O::sub(fxx, O::mul(fx, fx));
    const double var_y = O::sub(fyy, O::mul(fy, fy));
    const double cov = O::sub(fxy, O::mul(fx, fy));
    const double num = O::mul(O::add(O::mul(O::mul(2.0, fx), fy), s.c1), O::add(O::mul(2.0, cov), s.c2));
    const double den =
        O::mul(O::add(O::add(O::mul(fx, fx), O::mul(fy, fy)), s.c1), O::add(O::add(var_x, var_y), s.c2));
    map[(long long)img * nout + e] = O::div(num, den);
}

// leaf sums of NumPy's pairwise summation: leaf t covers [off[t], off[t]+len[t])
// of image blockIdx.y's map (len <= 128)
__global__ void __launch_bounds__(256) k_pairwise_leaves(const double* __restrict__ map, long long nper,
                                                         const long long* __restrict__ off,
                                                         const int* __restrict__ len, int nleaves, double* out) {
    pdl_sync();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nleaves) return;
    const double* a = map + (long long)blockIdx.y * nper + off[t];
    const int n = len[t];
    double res;
    if (n < 8) {
        res = -0.0;
        for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    } else {
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    }
    out[(long long)blockIdx.y * nleaves + t] = res;
}

}  // namespace cmg
