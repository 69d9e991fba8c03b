/*
 * cmg_oracle.c -- CPU restatement of the reference multigrid curvature
 * V-cycle (arXiv 2204.07921, package `curvemg`).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path (paper_2204_07921_b200 + libcmg.so)
 * never links or calls it.
 *
 * It restates, scalar and in plain C, the NumPy operation sequence of the
 * reference so that results are bit-identical (IEEE binary64, round to
 * nearest, no FMA contraction: build with -ffp-contract=off):
 *
 *   solver_pad            tangent.py:262-269  (np.pad reflect/odd, incl. the
 *                                              iterated and singleton cases of
 *                                              numpy's _set_reflect_both)
 *   distance_fields       tangent.py:272-310
 *   curvature_field       tangent.py:313-325
 *   energy                tangent.py:328-341
 *   backward_step         fbs.py:84-90, StepSchedule.eta fbs.py:68-72
 *   color_corrections     driver.py:175-222
 *   sweep_layer           driver.py:225-251
 *   layer_sequence        driver.py:254-258
 *   denoise               driver.py:261-314
 *   rel_err_energy        driver.py:146-150, _rel_u_guarded driver.py:161-166
 *
 * NumPy reduction orders reproduced (probed on NumPy 2.3.5):
 *   - x.sum() of a contiguous array: pairwise over the flattened array
 *     (blocks of 8 accumulators, recursive halving above 128 elements).
 *   - d.mean(axis=0) over planes: sequential in plane order, except when the
 *     colour class holds exactly one patch (then pairwise over the planes).
 *   - blocks.mean(axis=(1,3)) for f*: per patch, rows summed sequentially,
 *     each row pairwise -- except when the colour class has a single patch
 *     column, where NumPy coalesces the patch into one flat pairwise sum.
 * The reference's per-band thread pool does not change these orders for
 * threads=1, which is the semantics restated here.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define MAX_LAYER 6
#define MAX_PLANES 256

typedef struct {
    int x0, x1, y0, y1, z0, z1;
    double ds2;
} plane_t;

static plane_t g_planes[MAX_LAYER + 1][MAX_PLANES];
static int g_nplanes[MAX_LAYER + 1];
static int g_planes_ready = 0;

static int igcd(int a, int b) {
    a = abs(a);
    b = abs(b);
    while (b) {
        int t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* floor division like Python's // for the gcd-normalised direction key */
static int pydiv(int a, int b) {
    int q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

typedef struct {
    int r, c;
    double ang;
} rep_t;

static int rep_cmp(const void* a, const void* b) {
    double x = ((const rep_t*)a)->ang, y = ((const rep_t*)b)->ang;
    return (x < y) ? -1 : (x > y) ? 1 : 0;
}

/* plane_set, tangent.py:95-133 */
static void build_planes(void) {
    if (g_planes_ready) return;
    for (int layer = 1; layer <= MAX_LAYER; ++layer) {
        int n = 0;
        if (layer > 1) {
            n = g_nplanes[layer - 1];
            memcpy(g_planes[layer], g_planes[layer - 1], sizeof(plane_t) * n);
        }
        int r = 1 << (layer - 1);
        rep_t reps[4 * 64 + 8];
        int nr = 0;
        for (int dr = -r; dr <= r; ++dr)
            for (int dc = -r; dc <= r; ++dc) {
                int ad = abs(dr) > abs(dc) ? abs(dr) : abs(dc);
                if (ad != r) continue;
                if (dr < 0 || (dr == 0 && dc > 0)) {
                    reps[nr].r = dr;
                    reps[nr].c = dc;
                    reps[nr].ang = atan2((double)(-dr), (double)dc);
                    nr++;
                }
            }
        qsort(reps, nr, sizeof(rep_t), rep_cmp);
        for (int i = 0; i < nr; ++i) {
            int pr = reps[i].r, pc = reps[i].c;
            int g = igcd(pr, pc);
            int kr = pydiv(pr, g), kc = pydiv(pc, g);
            int dup = 0;
            for (int k = 0; k < n; ++k) {
                int gg = igcd(g_planes[layer][k].x0, g_planes[layer][k].x1);
                if (pydiv(g_planes[layer][k].x0, gg) == kr && pydiv(g_planes[layer][k].x1, gg) == kc) {
                    dup = 1;
                    break;
                }
            }
            if (dup) continue;
            int qr = -pc, qc = pr; /* rot90 */
            double ds2 = (double)(pr * pr + pc * pc);
            plane_t a = {pr, pc, qr, qc, -pr, -pc, ds2};
            plane_t b = {pr, pc, -pr, -pc, -qr, -qc, ds2};
            g_planes[layer][n++] = a;
            g_planes[layer][n++] = b;
        }
        g_nplanes[layer] = n;
    }
    g_planes_ready = 1;
}

int orc_plane_table(int layer, int* out6, double* ds2) {
    build_planes();
    if (layer < 1 || layer > MAX_LAYER) return -1;
    for (int i = 0; i < g_nplanes[layer]; ++i) {
        const plane_t* p = &g_planes[layer][i];
        out6[6 * i + 0] = p->x0;
        out6[6 * i + 1] = p->x1;
        out6[6 * i + 2] = p->y0;
        out6[6 * i + 3] = p->y1;
        out6[6 * i + 4] = p->z0;
        out6[6 * i + 5] = p->z1;
        if (ds2) ds2[i] = p->ds2;
    }
    return g_nplanes[layer];
}

/* ---------------------------------------------------------------------- */
/* NumPy pairwise summation (numpy/_core/src/umath/loops_utils.h.src)      */
/* ---------------------------------------------------------------------- */
static double pairwise_sum(const double* a, long n, long stride) {
    if (n < 8) {
        double res = -0.0;
        for (long i = 0; i < n; ++i) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int t = 0; t < 8; ++t) r[t] = a[t * stride];
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int t = 0; t < 8; ++t) r[t] += a[(i + t) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    } else {
        long n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2, stride) + pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

double orc_pairwise_sum(const double* a, long n) { return pairwise_sum(a, n, 1); }

/* ---------------------------------------------------------------------- */
/* np.pad(a, ((t,b),(l,r)), mode="reflect", reflect_type="odd")           */
/* ---------------------------------------------------------------------- */

/* One axis of numpy's iterative reflect padding on a 1-D strided line of
 * total length L = left + len + right (numpy _set_reflect_both loop).  */
static void reflect_line(double* line, long stride, int left, int len, int right) {
    if (len == 1) { /* singleton: legacy 'edge' behaviour */
        double e = line[(long)left * stride];
        for (int i = 0; i < left; ++i) line[(long)i * stride] = e;
        for (int i = 0; i < right; ++i) line[(long)(left + 1 + i) * stride] = e;
        return;
    }
    int total = left + len + right;
    int lp = left, rp = right;
    while (lp > 0 || rp > 0) {
        int old_length = total - rp - lp;
        old_length = ((old_length - 1) / (len - 1)) * (len - 1) + 1;
        old_length -= 1;
        if (lp > 0) {
            int chunk = old_length < lp ? old_length : lp;
            /* left_chunk = padded[lp+chunk : lp : -1]  -> indices lp+chunk .. lp+1 */
            double edge = line[(long)lp * stride];
            /* write into [lp-chunk, lp): element j (0..chunk-1) of the
               inserted slice = 2*edge - padded[lp+chunk-j] */
            double tmp[4096];
            for (int j = 0; j < chunk; ++j) tmp[j] = 2.0 * edge - line[(long)(lp + chunk - j) * stride];
            for (int j = 0; j < chunk; ++j) line[(long)(lp - chunk + j) * stride] = tmp[j];
            lp -= chunk;
        }
        if (rp > 0) {
            int chunk = old_length < rp ? old_length : rp;
            /* start = -rp - 2 (python negative index), step -1, chunk elems */
            int start = total - rp - 2;
            double edge = line[(long)(total - rp - 1) * stride];
            double tmp[4096];
            for (int j = 0; j < chunk; ++j) tmp[j] = 2.0 * edge - line[(long)(start - j) * stride];
            int dst = total - rp;
            for (int j = 0; j < chunk; ++j) line[(long)(dst + j) * stride] = tmp[j];
            rp -= chunk;
        }
    }
}

/* out has shape (m+t+b) x (n+l+r), row-major */
void orc_pad_odd(const double* a, int m, int n, int t, int b, int l, int r, double* out) {
    int M = m + t + b, N = n + l + r;
    for (int i = 0; i < M * N; ++i) out[i] = 0.0;
    for (int i = 0; i < m; ++i) memcpy(out + (long)(t + i) * N + l, a + (long)i * n, sizeof(double) * n);
    /* axis 0: columns restricted to the original column range */
    if (t > 0 || b > 0)
        for (int k = l; k < l + n; ++k) reflect_line(out + k, N, t, m, b);
    /* axis 1: every (padded) row */
    if (l > 0 || r > 0)
        for (int i = 0; i < M; ++i) reflect_line(out + (long)i * N, 1, l, n, r);
}

/* ---------------------------------------------------------------------- */
/* Level geometry (hierarchy.py:29-73)                                     */
/* ---------------------------------------------------------------------- */
typedef struct {
    int layer, side, r, mj, nj, mp, np_;
} level_t;

static level_t make_level(int m, int n, int layer) {
    level_t L;
    L.layer = layer;
    L.side = (1 << layer) - 1;
    L.r = 1 << (layer - 1);
    L.mj = (m + L.side - 1) / L.side;
    L.nj = (n + L.side - 1) / L.side;
    L.mp = L.mj * L.side;
    L.np_ = L.nj * L.side;
    return L;
}

/* perpendicular and vertical distance of one plane, tangent.py:296-309 */
static inline void plane_dist(const double* up, long W, long cidx, const plane_t* pl, double* perp,
                              double* vert) {
    double ux = up[cidx + pl->x0 * W + pl->x1];
    double uy = up[cidx + pl->y0 * W + pl->y1];
    double uz = up[cidx + pl->z0 * W + pl->z1];
    double uo = up[cidx];
    double p = uy - ux;
    double q = uz - ux;
    int dy0 = pl->y0 - pl->x0, dy1 = pl->y1 - pl->x1;
    int dz0 = pl->z0 - pl->x0, dz1 = pl->z1 - pl->x1;
    double nx = (double)dz1 * p - (double)dy1 * q;
    double ny = (double)dy0 * q - (double)dz0 * p;
    int nz = dz0 * dy1 - dz1 * dy0;
    double raw = (double)(-pl->x0) * nx - (double)pl->x1 * ny + (double)nz * (uo - ux);
    if (vert) *vert = raw / (double)(-nz);
    if (perp) *perp = raw / sqrt((nx * nx + ny * ny) + (double)(nz * nz));
}

/* f* of one patch from the diff snapshot (driver.py:244-246) */
static double patch_fstar(const double* diff, long W, long r0, long c0, int s, int flat) {
    /* diff is the full padded diff, patch top-left at (1+r0, 1+c0) */
    double acc;
    if (flat) {
        /* NumPy coalesces the (s, s) block into one pairwise reduction */
        double buf[63 * 63];
        for (int a = 0; a < s; ++a)
            for (int b = 0; b < s; ++b) buf[a * s + b] = diff[(1 + r0 + a) * W + 1 + c0 + b];
        acc = 0.0 + pairwise_sum(buf, (long)s * s, 1);
    } else {
        acc = 0.0;
        for (int a = 0; a < s; ++a) acc = acc + pairwise_sum(diff + (1 + r0 + a) * W + 1 + c0, s, 1);
    }
    return acc / (double)(s * s);
}

/* sweep_layer, driver.py:225-251 (u is m x n, updated in place) */
static int sweep_layer_impl(double* u, const double* fpad, int m, int n, level_t L, int mode,
                            int inner_iters, double alpha, int nthreads) {
    build_planes();
    const plane_t* pls = g_planes[L.layer];
    const int iota = g_nplanes[L.layer];
    const int s = L.side;
    const long H = L.mp + 2, W = L.np_ + 2;
    const int bpad = 1 + L.mp - m, rpad = 1 + L.np_ - n;
    double* upad = (double*)malloc(sizeof(double) * H * W);
    double* diff = (double*)malloc(sizeof(double) * H * W);
    double* cbuf = (double*)malloc(sizeof(double) * (size_t)L.mj * L.nj);
    int nonfinite = 0;
    static const int order[4][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}};
    /* backward-step constants (Python float arithmetic) */
    double wt[16], den[16];
    for (int t = 0; t < inner_iters; ++t) {
        double eta = (t == 0) ? 1.0 : 1.0 / sqrt((double)t);
        wt[t] = alpha * eta * (double)(s * s);
        den[t] = 2.0 + wt[t];
    }
    (void)nthreads;
    for (int ci = 0; ci < 4; ++ci) {
        int p = order[ci][0], q = order[ci][1];
        orc_pad_odd(u, m, n, 1, bpad, 1, rpad, upad);
        for (long i = 0; i < H * W; ++i) diff[i] = fpad[i] - upad[i];
        int hc = (L.mj - p + 1) / 2, wc = (L.nj - q + 1) / 2;
        if (hc <= 0 || wc <= 0) continue;
        int flat = (wc == 1);
        int single = (hc * wc == 1);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) if (nthreads > 1)
#endif
        for (int a = 0; a < hc; ++a) {
            double dv[MAX_PLANES], vv[MAX_PLANES];
            for (int b = 0; b < wc; ++b) {
                int i1 = 2 * a + p, i2 = 2 * b + q;
                long r0 = (long)i1 * s, c0 = (long)i2 * s;
                double fstar = patch_fstar(diff, W, r0, c0, s, flat);
                long cidx = (1 + r0 + L.r - 1) * W + (1 + c0 + L.r - 1);
                double chalf;
                if (mode == 0) {
                    for (int k = 0; k < iota; ++k) plane_dist(upad, W, cidx, &pls[k], &dv[k], NULL);
                    double sum;
                    if (single) {
                        sum = pairwise_sum(dv, iota, 1);
                    } else {
                        sum = dv[0];
                        for (int k = 1; k < iota; ++k) sum = sum + dv[k];
                    }
                    chalf = sum / (double)iota;
                } else {
                    for (int k = 0; k < iota; ++k) plane_dist(upad, W, cidx, &pls[k], NULL, &vv[k]);
                    int imin = 0, imax = 0;
                    /* np.argmin / np.argmax: first index; first NaN wins */
                    if (!isnan(vv[0])) {
                        for (int k = 1; k < iota; ++k) {
                            if (isnan(vv[k])) { imin = k; break; }
                            if (vv[k] < vv[imin]) imin = k;
                        }
                        for (int k = 1; k < iota; ++k) {
                            if (isnan(vv[k])) { imax = k; break; }
                            if (vv[k] > vv[imax]) imax = k;
                        }
                    }
                    int star = (fabs(vv[imin]) <= fabs(vv[imax])) ? imin : imax;
                    plane_dist(upad, W, cidx, &pls[star], &chalf, NULL);
                }
                double c = 0.0;
                for (int t = 0; t < inner_iters; ++t) c = ((c + chalf) + wt[t] * fstar) / den[t];
                cbuf[(long)i1 * L.nj + i2] = c;
            }
        }
        /* prolongate (hierarchy.py:117-126) + u += ... (driver.py:249-251) */
        for (int a = 0; a < hc; ++a)
            for (int b = 0; b < wc; ++b) {
                int i1 = 2 * a + p, i2 = 2 * b + q;
                double c = cbuf[(long)i1 * L.nj + i2];
                if (!isfinite(c)) nonfinite = 1;
            }
        if (nonfinite) break;
        for (int a = 0; a < hc; ++a)
            for (int b = 0; b < wc; ++b) {
                int i1 = 2 * a + p, i2 = 2 * b + q;
                double c = cbuf[(long)i1 * L.nj + i2];
                for (int rr = i1 * s; rr < (i1 + 1) * s && rr < m; ++rr)
                    for (int cc = i2 * s; cc < (i2 + 1) * s && cc < n; ++cc) u[(long)rr * n + cc] += c;
            }
    }
    free(upad);
    free(diff);
    free(cbuf);
    return nonfinite ? 1 : 0;
}

static double* make_fpad(const double* f, int m, int n, level_t L) {
    double* fp = (double*)malloc(sizeof(double) * (size_t)(L.mp + 2) * (L.np_ + 2));
    orc_pad_odd(f, m, n, 1, 1 + L.mp - m, 1, 1 + L.np_ - n, fp);
    return fp;
}

/* Public: one level visit (driver.sweep_layer). returns 0 ok, 1 non-finite correction. */
int orc_sweep_layer(double* u, const double* f, int m, int n, int layer, int mode, int inner_iters,
                    double alpha, int nthreads) {
    if (layer < 1 || layer > MAX_LAYER || m < 1 || n < 1) return -1;
    level_t L = make_level(m, n, layer);
    double* fp = make_fpad(f, m, n, L);
    int rc = sweep_layer_impl(u, fp, m, n, L, mode, inner_iters, alpha, nthreads);
    free(fp);
    return rc;
}

/* curvature_field + energy, tangent.py:313-341 */
double orc_curvature_sum(const double* u, int m, int n, int mode, double* field_out) {
    build_planes();
    double* up = (double*)malloc(sizeof(double) * (size_t)(m + 2) * (n + 2));
    orc_pad_odd(u, m, n, 1, 1, 1, 1, up);
    double* fld = field_out ? field_out : (double*)malloc(sizeof(double) * (size_t)m * n);
    const long W = n + 2;
    for (int i = 0; i < m; ++i)
        for (int k = 0; k < n; ++k) {
            long cidx = (long)(i + 1) * W + (k + 1);
            double kmin = 0, kmax = 0;
            int nan = 0;
            for (int l = 0; l < 8; ++l) {
                double v;
                plane_dist(up, W, cidx, &g_planes[1][l], NULL, &v);
                double kap = v / g_planes[1][l].ds2;
                if (isnan(kap)) nan = 1;
                if (l == 0) {
                    kmin = kap;
                    kmax = kap;
                } else {
                    if (kap < kmin) kmin = kap;
                    if (kap > kmax) kmax = kap;
                }
            }
            double val = (mode == 0) ? fabs(0.5 * (kmin + kmax)) : fabs(kmin * kmax);
            fld[(long)i * n + k] = nan ? NAN : val;
        }
    double s = pairwise_sum(fld, (long)m * n, 1);
    free(up);
    if (!field_out) free(fld);
    return s;
}

double orc_energy(const double* u, const double* f, int m, int n, double alpha, int mode) {
    double curv = orc_curvature_sum(u, m, n, mode, NULL);
    double* d = (double*)malloc(sizeof(double) * (size_t)m * n);
    for (long i = 0; i < (long)m * n; ++i) {
        double t = u[i] - f[i];
        d[i] = t * t;
    }
    double fid = 0.5 * alpha * pairwise_sum(d, (long)m * n, 1);
    free(d);
    return curv + fid;
}

static double rel_err_energy(double fnew, double fold) {
    if (fnew == 0.0) return fabs(fold);
    return fabs(fnew - fold) / fabs(fnew);
}

/*
 * denoise, driver.py:261-314.  Traces have room for max_outer+1 entries.
 * Returns 0 converged, 2 not converged, 3 divergence (non-finite energy),
 * 1 non-finite correction (prolongate ValueError), -1 bad args.
 */
int orc_denoise(const double* f, int m, int n, double alpha, int mode, int layers, double epsilon,
                int max_outer, int inner_iters, int stop_rule, int full_vcycle, const double* ref,
                double peak, int nthreads, double* u_out, double* energy, double* rel_e,
                double* rel_u, double* psnr, int* iterations) {
    if (layers < 1 || layers > MAX_LAYER || m < 1 || n < 1) return -1;
    long N = (long)m * n;
    level_t Ls[MAX_LAYER + 1];
    double* fps[MAX_LAYER + 1];
    for (int j = 1; j <= layers; ++j) {
        Ls[j] = make_level(m, n, j);
        fps[j] = make_fpad(f, m, n, Ls[j]);
    }
    int seq[2 * MAX_LAYER];
    int nseq = 0;
    for (int j = 1; j <= layers; ++j) seq[nseq++] = j;
    if (full_vcycle)
        for (int j = layers - 1; j >= 1; --j) seq[nseq++] = j;
    double* u = u_out;
    memcpy(u, f, sizeof(double) * N);
    double* uprev = (double*)malloc(sizeof(double) * N);
    double* tmp = (double*)malloc(sizeof(double) * N);
    int status = 2;
#define PSNR_AT(idx)                                                                 \
    do {                                                                             \
        if (ref && psnr) {                                                           \
            for (long i_ = 0; i_ < N; ++i_) {                                        \
                double d_ = u[i_] - ref[i_];                                         \
                tmp[i_] = d_ * d_;                                                   \
            }                                                                        \
            double mse_ = pairwise_sum(tmp, N, 1) / (double)N;                       \
            psnr[idx] = (mse_ == 0.0) ? INFINITY : 10.0 * log10(peak * peak / mse_); \
        }                                                                            \
    } while (0)
    double fval = orc_energy(u, f, m, n, alpha, mode);
    energy[0] = fval;
    rel_e[0] = NAN;
    rel_u[0] = NAN;
    PSNR_AT(0);
    int it = 0;
    for (int outer = 1; outer <= max_outer; ++outer) {
        memcpy(uprev, u, sizeof(double) * N);
        double fprev = fval;
        int bad = 0;
        for (int si = 0; si < nseq && !bad; ++si) {
            int j = seq[si];
            bad = sweep_layer_impl(u, fps[j], m, n, Ls[j], mode, inner_iters, alpha, nthreads);
        }
        if (bad) {
            status = 1;
            it = outer - 1;
            break;
        }
        fval = orc_energy(u, f, m, n, alpha, mode);
        it = outer;
        if (!isfinite(fval)) {
            energy[outer] = fval;
            status = 3;
            break;
        }
        double re = rel_err_energy(fval, fprev);
        for (long i = 0; i < N; ++i) tmp[i] = fabs(u[i] - uprev[i]);
        double num = pairwise_sum(tmp, N, 1);
        for (long i = 0; i < N; ++i) tmp[i] = fabs(u[i]);
        double den = pairwise_sum(tmp, N, 1);
        double ru = (den == 0.0) ? ((num == 0.0) ? 0.0 : INFINITY) : num / den;
        energy[outer] = fval;
        rel_e[outer] = re;
        rel_u[outer] = ru;
        PSNR_AT(outer);
        double crit = (stop_rule == 0) ? re : ru;
        if (crit <= epsilon) {
            status = 0;
            break;
        }
    }
#undef PSNR_AT
    *iterations = it;
    for (int j = 1; j <= layers; ++j) free(fps[j]);
    free(uprev);
    free(tmp);
    return status;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
