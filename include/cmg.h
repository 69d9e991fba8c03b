/*
 * cmg.h -- C ABI of the B200 multigrid curvature-energy solver (libcmg.so).
 *
 * Drop-in boundary for the reference package `curvemg` (arXiv 2204.07921).
 * The reference has no FFI: its boundary is the Python call
 *     curvemg.denoise(f: Image, config: SolverConfig, reference=None)
 *         -> (Image, ConvergenceTrace)
 * (/root/reference/pkg/src/curvemg/driver.py:261-314, re-exported at
 * __init__.py:3-10).  Each entry point below names the reference function it
 * replaces; the Python shim paper_2204_07921_b200.driver binds them through
 * ctypes and keeps the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *  - plain pointers and sizes only; images are row-major, batch x m x n,
 *    element type double (CMG_F64) or float (CMG_F32) as chosen at plan time;
 *  - every function returns a status code; cmg_last_error() gives the
 *    message of the last failure on the calling thread;
 *  - the caller owns host buffers, the plan owns device buffers, its CUDA
 *    stream and its CUDA graphs.  One plan per host thread; calls are
 *    synchronous with respect to the caller.
 */
#ifndef CMG_H
#define CMG_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define CMG_OK 0
#define CMG_EINVAL 1        /* ValueError: SolverConfig / Image validation (driver.py:56-72, image.py:51-58) */
#define CMG_NOT_CONVERGED 2 /* ran max_outer cycles without meeting epsilon (trace.converged == False) */
#define CMG_DIVERGED 3      /* SolverDivergence: non-finite energy (driver.py:302-303) */
#define CMG_ECUDA 4         /* CUDA runtime failure */
#define CMG_ENONFINITE 5    /* ValueError("corrections must be finite") (hierarchy.py:122-123) */

/* plan options */
#define CMG_MODE_MEAN 0  /* SolverConfig.mode == "mean"     (driver.py:47) */
#define CMG_MODE_GAUSS 1 /* SolverConfig.mode == "gaussian" */
#define CMG_F64 0
#define CMG_F32 1
#define CMG_PREC_EXACT 0 /* NumPy operation order, bit-identical to the reference in fp64 */
#define CMG_PREC_FAST 1  /* closed-form pair distances + rsqrt (mean mode only) */
#define CMG_STOP_REL_ENERGY 0
#define CMG_STOP_REL_U 1

typedef struct cmg_plan cmg_plan;

/* library version (major*10000 + minor*100 + patch) */
int cmg_version(void);

typedef struct cmg_mplan cmg_mplan;
typedef struct cmg_radon cmg_radon;

/* message of the last error on this thread ("" if none) */
const char* cmg_last_error(void);

/* number of visible CUDA devices */
int cmg_device_count(int* count);

/*
 * Create a solver plan for `batch` images of m x n pixels with `layers`
 * levels (hierarchy.build_hierarchy, hierarchy.py:83-91: 1 <= layers <= 6).
 * Replaces the per-call setup at the top of driver.denoise (driver.py:267-276).
 */
int cmg_plan_create(cmg_plan** out, int m, int n, int batch, int layers, int mode, int dtype, int precision,
                    int device);
int cmg_plan_destroy(cmg_plan* plan);

/*
 * Solve from HOST buffers (driver.denoise, driver.py:261-314).
 *   f_host        batch*m*n input images (element type of the plan)
 *   ref_host      optional clean images for the per-cycle PSNR (NULL: no PSNR)
 *   u_host_out    batch*m*n restored images
 *   alpha..peak   SolverConfig fields (driver.py:45-53) and Image.peak
 *   energy, rel_energy, rel_u, psnr, seconds
 *                 optional (NULL) trace outputs, batch x (max_outer+1)
 *                 doubles each (TraceRecord fields, driver.py:83-91)
 *   iterations    batch ints: ConvergenceTrace.iterations
 *   status        batch ints: CMG_OK (converged), CMG_NOT_CONVERGED,
 *                 CMG_DIVERGED or CMG_ENONFINITE per image
 * Returns CMG_OK if every image converged, otherwise the first non-OK
 * per-image status (or CMG_EINVAL / CMG_ECUDA).
 */
int cmg_solve(cmg_plan* plan, const void* f_host, const void* ref_host, void* u_host_out, double alpha,
              double epsilon, int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak,
              double* energy, double* rel_energy, double* rel_u, double* psnr, double* seconds, int* iterations,
              int* status);

/*
 * Same as cmg_solve with DEVICE pointers (inputs already resident in HBM).
 * Trace outputs are still host pointers.
 */
int cmg_solve_device(cmg_plan* plan, const void* f_dev, const void* ref_dev, void* u_dev_out, double alpha,
                     double epsilon, int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak,
                     double* energy, double* rel_energy, double* rel_u, double* psnr, double* seconds,
                     int* iterations, int* status);

/*
 * One level visit -- the four colour sweeps of driver.sweep_layer
 * (driver.py:225-251) -- on host buffers: u_host (batch*m*n) is updated in
 * place, f_host is the noisy input.  Parity-test entry point.
 */
int cmg_sweep_layer(cmg_plan* plan, void* u_host, const void* f_host, int layer, double alpha, int inner_iters);

/* tangent.energy (tangent.py:328-341) for each image: energy_out[batch] */
int cmg_energy(cmg_plan* plan, const void* u_host, const void* f_host, double alpha, double* energy_out);

/* tangent.plane_set (tangent.py:95-133) as compiled into the kernels:
 * writes count*6 ints (x0,x1,y0,y1,z0,z1) and count ds2 values; returns count. */
int cmg_plane_table(int layer, int* offsets, double* ds2);

/* Launch statistics of the last solve: number of kernels launched (all
 * nodes executed, including early-exit ones) and cycles executed. */
int cmg_plan_stats(cmg_plan* plan, long long* kernel_launches, int* cycles_run, double* device_ms);

/*
 * Time one sweep kernel with CUDA events on the plan's stream:
 * `reps` launches of the level-`layer` colour-`color` kernel (color < 0: all
 * four colours of the level; layer 0: the energy + finalize kernel) on the
 * data left by the last solve.  Writes the mean duration per launch in
 * milliseconds.  Used by bench.py's roofline.
 */
int cmg_time_sweep(cmg_plan* plan, int layer, int color, int reps, double* ms_per_launch);

/*
 * Building blocks for host-driven decompositions (horizontal strips over
 * several GPUs, paper_2204_07921_b200/strips.py).  A plan owns five device
 * buffers: 0..2 = the u rotation buffers, 3 = f, 4 = reference image; index
 * 5 is the batch x 6 doubles of cmg_strip_partials_async.
 */
/* device pointer of buffer `index` (batch*m*n elements) */
int cmg_plan_buffer(cmg_plan* plan, int index, void** dev_ptr);
/* whole-buffer host->device / device->host copies */
int cmg_buffer_upload(cmg_plan* plan, int index, const void* host);
int cmg_buffer_download(cmg_plan* plan, int index, void* host);
/* one level visit (driver.sweep_layer, driver.py:225-251) reading buffer
 * in_index and writing buffer out_index (distinct, 0..2) */
int cmg_level_step(cmg_plan* plan, int layer, int in_index, int out_index, double alpha, int inner_iters);
/* raw energy sums over rows [row_lo,row_hi) of every image: out[batch][5] =
 * {sum curvature (tangent.py:313-325), sum (u-f)^2, sum |u-u_prev|, sum |u|,
 *  sum (u-ref)^2}; F = s0 + (alpha/2) s1 as in tangent.energy (tangent.py:339-341) */
int cmg_energy_partials(cmg_plan* plan, int u_index, int prev_index, int use_ref, int row_lo, int row_hi,
                        double* out);

/*
 * Asynchronous strip cycle (one host synchronisation per V-cycle): everything
 * below only ENQUEUES on the plan's CUDA stream (cmg_plan_stream), so ghost-row
 * exchanges and all-reduces issued on that stream (NCCL / P2P copies) order
 * behind the level steps without host round trips.
 *   cmg_strip_begin           backward-step constants + per-image state reset
 *   cmg_level_step_async      cmg_level_step without the synchronisation
 *   cmg_strip_partials_async  energy sums of rows [row_lo,row_hi) -> device
 *                             buffer 5: batch x 5 sums, then batch
 *                             non-finite-correction flags (6 doubles for one
 *                             image; all-reduce it in place)
 *   cmg_strip_read            device buffer 5 -> host (6 x batch doubles), synchronises
 */
int cmg_plan_stream(cmg_plan* plan, void** stream);

/*
 * Multi-device batch plan: a batch of same-shape images sharded data-parallel
 * over n_devices GPUs (device_ids; an id may repeat: independent plans on one
 * GPU).  Device d gets a contiguous slice of images (sizes differ by <= 1);
 * cmg_mplan_solve runs the shards concurrently (one host thread per shard,
 * no collective: images are independent) with cmg_solve's arguments and
 * output layout for the WHOLE batch, and returns the first non-OK status
 * in image order.  The reference parallelises inside denoise
 * (driver.py:279-280); this is the library-level equivalent for batches.
 */
int cmg_mplan_create(cmg_mplan** out, int m, int n, int batch, int layers, int mode, int dtype, int precision,
                     const int* device_ids, int n_devices);
int cmg_mplan_destroy(cmg_mplan* mplan);
int cmg_mplan_solve(cmg_mplan* mplan, const void* f_host, const void* ref_host, void* u_host_out, double alpha,
                    double epsilon, int max_outer, int inner_iters, int stop_rule, int full_vcycle, double peak,
                    double* energy, double* rel_energy, double* rel_u, double* psnr, double* seconds, int* iterations,
                    int* status);
int cmg_strip_begin(cmg_plan* plan, double alpha, int inner_iters);
int cmg_level_step_async(cmg_plan* plan, int layer, int in_index, int out_index);
int cmg_strip_partials_async(cmg_plan* plan, int u_index, int prev_index, int use_ref, int row_lo, int row_hi);
int cmg_strip_read(cmg_plan* plan, double* out);

/*
 * curvemg.image.ssim (image.py:152-192) on the GPU, bit-identical: mean SSIM
 * of batch image pairs (batch*m*n row-major, dtype 0 f64 / 1 f32, values
 * taken as float64), 11x11 Gaussian windows.  The caller passes the window
 * (_gaussian_window(11, 1.5), image.py:157-160) and c1 = (0.01 peak)^2,
 * c2 = (0.03 peak)^2 computed as the reference does.  out[batch].
 */
int cmg_ssim_batch(int batch, int m, int n, int dtype, const void* a_host, const void* b_host, const double* window,
                   double c1, double c2, double* out);
/* the same on two of a plan's device buffers (0..2 u rotation, 3 f, 4 reference) */
int cmg_plan_ssim(cmg_plan* plan, int a_index, int b_index, const double* window, double c1, double c2, double* out);

/* Pinned host memory helpers (for host<->device copies at full PCIe rate). */
void* cmg_host_alloc(unsigned long long bytes);
int cmg_host_free(void* p);

/*
 * Measurement helper (no reference counterpart): L2 read bandwidth of the
 * device, the roofline denominator of L2-resident workloads (1024^2 fp64:
 * u and f = 16 MiB).  Streams a `bytes`-sized buffer (<< 126 MB L2, e.g.
 * 32 MiB) `reps` times with 16-byte loads from every SM (grid = SMs x 8 CTAs)
 * after one warm-up pass; *gbs = bytes * reps / elapsed (CUDA events).
 */
int cmg_l2_read_bandwidth(int device, long long bytes, int reps, double* gbs);

/*
 * Measurement helper (no reference counterpart): the FP64 pipe of the device,
 * the compute roof of the fp64 exact level-1 kernel.  *dfma_per_clk_per_sm =
 * sustained thread-level DFMAs per clock and SM (64 warps per SM, 8
 * independent chains per thread, CUDA events, nominal SM clock), *tflops the
 * same as 2 x DFMA/s, *dep_latency_cycles = clocks per DFMA of one dependent
 * chain in one warp (clock64).
 */
int cmg_fp64_probe(int device, double* dfma_per_clk_per_sm, double* dep_latency_cycles, double* tflops);

/*
 * Self test (no reference counterpart) of the branch-free correctly rounded
 * fp64 sqrt / div that the level-1 exact kernel uses (csrc/cmg_l1loop.cuh)
 * against the device library's sqrt.rn / div.rn on n host operand pairs:
 * out[0] / out[1] = in-range sqrt(a[i]) / (a[i] / b[i]) results that differ
 * from the library (must be 0), out[2] / out[3] = operands whose range test
 * selects the library path.
 */
int cmg_selftest_exact(int device, const double* a_host, const double* b_host, long long n,
                       unsigned long long* out);

/*
 * Curvature-regularised reconstruction (curvemg.reconstruction, fp64, device
 * pointers, work enqueued on `stream`; paper_2204_07921_b200.recon drives
 * them).  Parallel-beam Radon operator (reconstruction.py:123-183): the
 * caller passes each pixel's lower detector bin i0 and upper-bin weight w
 * per angle (n_angles x m*n, computed as the reference does); forward and
 * adjoint are bit-identical to the reference's bincount / gather.
 */
int cmg_radon_create(cmg_radon** out, int m, int n, int n_angles, int detector_count, double pixel_size,
                     const int* i0, const double* w, int device);
int cmg_radon_destroy(cmg_radon* radon);
int cmg_radon_forward(cmg_radon* radon, const double* x_dev, double* sino_dev, void* stream);
int cmg_radon_adjoint(cmg_radon* radon, const double* y_dev, double* x_dev, void* stream);
/* mean perpendicular plane distance at the patch centres of colour (p,q) of
 * level `layer` (reconstruction.py:403-404; hc*wc outputs, row-major) */
int cmg_recon_chalf(const double* u_dev, int m, int n, int layer, int p, int q, double* d_dev, void* stream);
/* u += prolongation of the colour's corrections c (reconstruction.py:410-413, :432) */
int cmg_recon_prolong(double* u_dev, const double* c_dev, int m, int n, int layer, int p, int q, void* stream);
/* per-patch sums of img over the colour's patches (reconstruction.py:415-419) */
int cmg_recon_block_sums(const double* img_dev, int m, int n, int layer, int p, int q, double* out_dev, void* stream);
/* level-1 mean-curvature mass, nblocks partial sums (tangent.curvature_field) */
int cmg_recon_curvature_partials(const double* u_dev, int m, int n, double* partial_dev, int nblocks, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CMG_H */
