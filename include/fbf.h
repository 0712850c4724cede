/*
 * fbf.h -- C ABI of the B200-native Fourier bilateral filtering stage
 * (arXiv 1811.02168), a drop-in for the reference fourierbf library's
 * filtering path (/root/reference/proj). Plain pointers and sizes only; no C++
 * or torch types cross this boundary, and no exception escapes it.
 *
 * Every entry point names the reference interface it replaces (file:line,
 * paths relative to /root/reference/proj). Status codes replace the
 * reference's exceptions; fbf_last_error() returns the message of the last
 * failure on the calling thread.
 *
 * Buffers: images are row-major, at(x, y) = pixels[y * width + x]
 * (include/fourierbf/image.hpp:25-26), single channel, float32 (the reference
 * uses double; the oracle widens float -> double exactly). Host buffers are
 * caller-owned; device buffers and streams are owned by a per-device context
 * inside the library.
 */
#ifndef FBF_H
#define FBF_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (exceptions in the reference) ------------------------- */
#define FBF_OK 0
#define FBF_EINVAL 1       /* std::invalid_argument (filter.cpp:132-134, kernels.cpp:13-14,106-107) */
#define FBF_ERANGE 2       /* pixel non-finite or outside [0, R] (filter.cpp:19-23) */
#define FBF_EUNREACHABLE 3 /* ToleranceUnreachable (approx.hpp:97-103); outputs hold the best fit */
#define FBF_ECUDA 4        /* CUDA runtime failure or no device */
#define FBF_ENOMEM 5
#define FBF_ECAPACITY 6    /* caller buffer too small / radius beyond the kernel's limit */

/* BorderPolicy (image.hpp:38), same order. */
#define FBF_BORDER_SYMMETRIC 0
#define FBF_BORDER_REPLICATE 1
#define FBF_BORDER_ZERO 2

/* RangeKernelKind (kernels.hpp:8), parametric kinds. */
#define FBF_KERNEL_GAUSSIAN 0
#define FBF_KERNEL_EXPONENTIAL 1
#define FBF_KERNEL_CAUCHY 2

/* Largest spatial radius ceil(3 theta) the fused sm_100a kernel is built for. */
#define FBF_MAX_RADIUS 32

/* Message of the last failed call on this thread ("" if none). */
const char* fbf_last_error(void);
/* Library / device info: number of visible CUDA devices (0 if none). */
int fbf_device_count(void);
/* Device used by the single-device host-buffer entry points
 * (fbf_fast_bilateral_f32, fbf_filter); default 0. One process per GPU sets
 * its local rank here. */
int fbf_set_device(int device);
int fbf_get_device(void);
/* Page-locked host buffers for the host-buffer entry points (cudaHostAlloc,
 * portable): pinned memory is what lets H2D/D2H of the pipelined calls run at
 * the PCIe rate. Pageable buffers work too, at the staged-copy rate. */
int fbf_host_alloc(size_t bytes, void** ptr);
int fbf_host_free(void* ptr);
/* Number of fused-kernel launches this process has issued (all devices). */
unsigned long long fbf_kernel_launches(void);

/* ---- L1 kernels: kernels.cpp ------------------------------------------- */
/* build_spatial_kernel (kernels.cpp:105-118): radius = ceil(3 theta); writes
 * 2*radius+1 unnormalised taps. Returns the radius, or -FBF_EINVAL /
 * -FBF_ECAPACITY (cap too small). */
int fbf_build_spatial_kernel(double theta, double* taps, int cap);
/* sample_range_kernel (kernels.cpp:78-103) for the parametric kinds:
 * values[2R+1] = phi(t - R), exactly symmetric. */
int fbf_sample_range_kernel(int kind, double sigma, int R, double* values);

/* ---- L2 approximation: approx.cpp (host, restated without Eigen) --------- */
/* nu = 2 pi / (2T+1) (approx.cpp:17-19). */
double fbf_frequency_of(int half_period);
/* fit_fixed_period (approx.cpp:105-117): least-squares c[K] at fixed (K, T);
 * err_out = ||A c - b||^2. samples has 2R+1 entries. */
int fbf_fit_fixed_period(const double* samples, int R, int K, int T, double* coeffs, double* err_out);
/* scan_period_errors (approx.cpp:119-130): errors[T-1] = E(K, T), T = 1..t_max. */
int fbf_scan_period_errors(const double* samples, int R, int K, int t_max, int threads, double* errors);
/* min_error_over_period (approx.cpp:132-144): ties keep the smaller T. */
int fbf_min_error_over_period(const double* samples, int R, int K, int t_max, int threads,
                              int* T_best, double* err_out);
/* optimize_parameters (approx.cpp:179-240), Algorithm 1. t_max<=0 -> 10R,
 * k_max<=0 -> 2R+1. Returns FBF_EUNREACHABLE with the best fit when no
 * K <= min(k_max, t_max+1) reaches tol. per_order (optional, 3*cap doubles)
 * receives (K, T_best, e(K)) rows; *n_orders their count. */
int fbf_optimize_parameters(const double* samples, int R, double tol, int t_max, int k_max,
                            int threads, int* K_out, int* T_out, double* coeffs, int coeff_cap,
                            double* err_out, double* per_order, int* n_orders);
/* CLI select_parameters (tools/fourierbf.cpp:185-234):
 *   eps>0, K=T=0      -> Algorithm 1 at tolerance eps
 *   K>0, T=0          -> best T over 1..10R, then fit
 *   K>0, T>0          -> fixed period
 *   method_fbf != 0   -> T = R with K given (or K* from eps)
 * eps together with K/T, or T without K, is FBF_EINVAL (as in the CLI). */
int fbf_select_params(int kind, double sigma, int R, double eps, int K, int T, int method_fbf,
                      int threads, int* K_out, int* T_out, double* coeffs, int coeff_cap,
                      double* err_out);

/* ---- L2 on the GPU: the period scan of approx.cpp:119-144 --------------- */
/* errors[(K - K_lo) * t_max + T - 1] = E(K, T) = ||A c - b||^2 for the nK
 * orders K_lo..K_lo+nK-1 and T = 1..t_max, FP64 on device `device`, one CTA
 * per (K, T) (fbf_scan.cu). Agrees with fbf_scan_period_errors to ~1e-15
 * relative near the minimum and ~1e-6 where A is ill-conditioned (tree
 * reductions), not bit for bit. FBF_ECAPACITY above
 * K = fbf_scan_gpu_max_order(R) (the design matrix lives in shared memory). */
int fbf_scan_period_errors_gpu(const double* samples, int R, int K_lo, int nK, int t_max, int device,
                               double* errors);
int fbf_scan_gpu_max_order(int R);
/* min_error_over_period (approx.cpp:132-144) through the GPU scan + exact
 * host re-check: the same (T_best, E) as fbf_min_error_over_period. */
int fbf_min_error_over_period_gpu(const double* samples, int R, int K, int t_max, int device, int* T_best,
                                  double* err_out);
/* fbf_optimize_parameters / fbf_select_params with the period scans on the
 * GPU: every T whose GPU error lies within a relative 1e-4 of the GPU minimum
 * is re-fitted with the host routine and the argmin of those exact errors is
 * taken (smaller T on ties), so K, T, the coefficients and the error equal
 * the host versions'. Orders above fbf_scan_gpu_max_order(R) scan on the host. */
int fbf_optimize_parameters_gpu(const double* samples, int R, double tol, int t_max, int k_max, int device,
                                int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out,
                                double* per_order, int* n_orders);
int fbf_select_params_gpu(int kind, double sigma, int R, double eps, int K, int T, int method_fbf, int device,
                          int* K_out, int* T_out, double* coeffs, int coeff_cap, double* err_out);
/* ---- L2 lookup table: lut.cpp -------------------------------------------- */
/* build_lut (lut.cpp:61-113): K*[i*n_eps+j], T*[i*n_eps+j] of Algorithm 1 for
 * the Gaussian kernel at (sigmas[i], epsilons[j]); grids strictly ascending
 * (sigma, log10(1/eps)), >= 2 points each, eps in (0,1). device >= 0: period
 * scans on that GPU (identical cells); device < 0: `threads` host threads.
 * A cell that cannot reach its tolerance fails the build, cell identified. */
int fbf_build_lut(const double* sigmas, int n_sigma, const double* epsilons, int n_eps, int R, int t_max,
                  int device, int threads, int* K_out, int* T_out);
/* query_lut (lut.cpp:116-143): bilinear in (sigma, log10(1/eps)), K rounded
 * up, T to nearest; outside the grid FBF_ERANGE (std::out_of_range). */
int fbf_query_lut(const double* sigma_grid, int n_sigma, const double* logeps_grid, int n_eps, const int* K,
                  const int* T, double sigma, double eps, int* K_out, int* T_out);
/* ---- L3 filter: filter.cpp (the hot path, sm_100a) ---------------------- */
/* StageTimings (include/fourierbf/filter.hpp:19-24), filled by accumulation
 * (+=) like filter.cpp:151-211. The kernel fuses channel generation,
 * convolutions and the combine, so their device time is reported as
 * convolution_seconds and auxiliary/combine stay 0; fit_seconds is left to the
 * caller (the reference's CLI fills it, tools/fourierbf.cpp:249-261). The
 * host-buffer call adds the busy time of its PCIe copies and its wall time. */
typedef struct fbf_stage_timings {
    double fit_seconds;
    double auxiliary_seconds;
    double convolution_seconds;  /* fused kernel launches, device time (CUDA events) */
    double combine_seconds;
    double h2d_seconds;          /* host -> device copies, device time */
    double d2h_seconds;          /* device -> host copies, device time */
    double wall_seconds;         /* the whole call on the host clock */
} fbf_stage_timings;

/* fast_bilateral (filter.hpp:43-46, filter.cpp:129-213) with the whole
 * FourierApproximation (approx.hpp:14-22): `frequency` is approx.frequency,
 * used as given like filter.cpp:139 (nu k f is the phase of term k); 0 means
 * frequency_of(T). timings (optional) as above. Everything else as
 * fbf_fast_bilateral_f32. */
int fbf_fast_bilateral_ex(const float* img, int width, int height, double theta, int K, int T, int R,
                          double frequency, const double* coeffs, int border, float* out, long long* fallbacks,
                          fbf_stage_timings* timings);
/* fast_bilateral (filter.hpp:43-46, filter.cpp:129-213) on HOST buffers:
 * validates intensities, copies img to the device, runs the fused kernel,
 * copies out back. K >= 1 coefficients c_0..c_{K-1}, T >= 1, R >= 1.
 * *fallbacks (optional) is INCREMENTED by the number of pixels whose
 * denominator was <= 1e-12 (FilterDiagnostics, filter.hpp:15-17). */
int fbf_fast_bilateral_f32(const float* img, int width, int height, double theta, int K, int T,
                           int R, const double* coeffs, int border, float* out,
                           long long* fallbacks);
/* Same, device-resident: d_img / d_out are device pointers on device `device`;
 * enqueued on `stream` (a cudaStream_t; NULL = the legacy default stream)
 * and returns without synchronising.
 * d_fallbacks (optional) is a device unsigned long long counter that is
 * atomically incremented. No intensity validation (use fbf_validate_f32). */
int fbf_fast_bilateral_f32_device(const float* d_img, int width, int height, double theta, int K,
                                  int T, int R, const double* coeffs, int border, float* d_out,
                                  unsigned long long* d_fallbacks, int device, void* stream);
/* Device-resident entry points take the scratch of multi-chunk plans (2K-1
 * channel pairs beyond one launch) from a stream-ordered pool on `stream`,
 * so concurrent calls on different streams never share buffers. They restore
 * the calling thread's current device before returning. */
/* Batch of n_frames independent frames (frame f at img + f*width*height),
 * sharded across the first n_gpus devices (0 -> all), one host thread each;
 * n_gpus = 1 uses the default device (fbf_set_device). Within a device the
 * frames are pipelined: H2D of later frames and D2H of earlier ones overlap
 * the kernels. Output frames land in disjoint slices of out. */
int fbf_fast_bilateral_batch_f32(const float* img, int n_frames, int width, int height,
                                 double theta, int K, int T, int R, const double* coeffs,
                                 int border, float* out, long long* fallbacks, int n_gpus);
/* One large image split into n_gpus row bands, each staged with replicated
 * ceil(3 theta)-row halos (border rows keep the mirror semantics); no
 * collective, outputs are disjoint row slices. Bit-identical to n_gpus = 1.
 * Each device pipelines its band (H2D / kernel / D2H in sub-bands); n_gpus = 1
 * uses the default device (fbf_set_device). */
int fbf_fast_bilateral_bands_f32(const float* img, int width, int height, double theta, int K,
                                 int T, int R, const double* coeffs, int border, float* out,
                                 long long* fallbacks, int n_gpus);
/* Device-resident band for one rank: d_src holds global rows
 * [src_row0, src_row0 + src_rows) of a width x height image (row pitch =
 * width) and must contain every row the border mapping reaches for output rows
 * [out_row0, out_row0 + out_rows); d_dst receives those output rows. Use
 * fbf_band_source_rows() to size the halo. */
int fbf_fast_bilateral_band_f32_device(const float* d_src, int src_row0, int src_rows,
                                       int width, int height, int out_row0, int out_rows,
                                       double theta, int K, int T, int R, const double* coeffs,
                                       int border, float* d_dst,
                                       unsigned long long* d_fallbacks, int device, void* stream);
/* Host-buffer band for one rank (one process per GPU): src holds global rows
 * [src_row0, src_row0 + src_rows) of a width x height image -- the rank's band plus
 * the halo fbf_band_source_rows() reports -- and out receives output rows
 * [out_row0, out_row0 + out_rows). Runs on the default device (fbf_set_device) with
 * the single-image call's H2D / kernel / D2H pipeline and in-kernel intensity
 * validation; bit-identical to the same rows of fbf_fast_bilateral_f32 on the whole
 * image (the band split of fbf_fast_bilateral_bands_f32, one band per process). */
int fbf_fast_bilateral_band_f32(const float* src, int src_row0, int src_rows, int width, int height,
                                int out_row0, int out_rows, double theta, int K, int T, int R,
                                const double* coeffs, int border, float* out, long long* fallbacks);
/* Device-resident batch: n_frames frames at d_img + f*width*height, one
 * launch on `stream` (CTAs share the (frame, strip, row) units evenly, so the
 * per-segment warm-up rows amortise over the batch). No validation. */
int fbf_fast_bilateral_batch_f32_device(const float* d_img, int n_frames, int width, int height, double theta, int K,
                                        int T, int R, const double* coeffs, int border, float* d_out,
                                        unsigned long long* d_fallbacks, int device, void* stream);
/* Global source-row window [*row0, *row0 + *rows) needed for output rows
 * [out_row0, out_row0 + out_rows) at radius ceil(3 theta). */
int fbf_band_source_rows(int height, int out_row0, int out_rows, double theta, int border,
                         int* row0, int* rows);
/* fast_bilateral on 8-bit host buffers (the CLI's PGM path: read_pgm,
 * imageio.cpp:53-80, widens bytes exactly). Exactly one output: out_u8
 * receives the result clamped to [0,255] and rounded half away from zero
 * (write_clamped + write_pgm, tools/fourierbf.cpp:71-76, imageio.cpp:83-89);
 * out_f32 the float result. 1 byte per pixel crosses PCIe each way instead of 4. */
int fbf_fast_bilateral_u8(const unsigned char* img, int width, int height, double theta, int K, int T, int R,
                          const double* coeffs, int border, unsigned char* out_u8, float* out_f32,
                          long long* fallbacks);
/* Convenience signature from the north star: parameters chosen on the host
 * like the CLI's `filter --eps` (eps_or_K < 1: tolerance) or `--K` (integer
 * eps_or_K >= 1: fixed K, T scanned over 1..10R); Gaussian range kernel,
 * R = 255, symmetric border. The period scans run on the GPU
 * (fbf_select_params_gpu: same K, T, c as the host scan). */
int fbf_filter(const float* img, int height, int width, double theta, double sigma,
               double eps_or_K, float* out);

/* validate_intensities (filter.cpp:19-23) on the device: returns FBF_OK or
 * FBF_ERANGE. */
int fbf_validate_f32_device(const float* d_img, size_t n, int R, int device, void* stream);

/* ---- L3 reference filter and metrics on the GPU (fbf_brute.cu) ---------- */
/* brute_bilateral (filter.cpp:83-127): the direct (2r+1)^2 bilateral filter
 * with the range kernel read from its lattice (range[2R+1], phi(t) =
 * range[t + R], t = lround(neighbour - centre)). FP64 with the reference's
 * operation order and no FMA contraction: on float32 inputs the output equals
 * the reference's compiled brute_bilateral bit for bit. out is double (the
 * reference's GrayImage). Radius ceil(3 theta) <= 64. */
int fbf_brute_bilateral_f32(const float* img, int width, int height, double theta, const double* range, int R,
                            int border, double* out, long long* fallbacks);
/* Same on device buffers (no intensity validation), enqueued on `stream`;
 * returns after the kernel finished. */
int fbf_brute_bilateral_f32_device(const float* d_img, int width, int height, double theta, const double* range,
                                   int R, int border, double* d_out, unsigned long long* d_fallbacks, int device,
                                   void* stream);
/* compare_images (metrics.cpp:10-26) of a double reference image and a float
 * candidate, both on the device: MSE, PSNR = 10 log10(255^2 / MSE) (+inf when
 * equal) and max |difference|. Deterministic (fixed reduction order). */
int fbf_compare_images_device(const double* d_ref, const float* d_cand, size_t n, double* mse, double* psnr_db,
                              double* max_abs, int device, void* stream);
/* ---- L4 synthetic inputs (synthetic.cpp + BASELINE.json generators) ------ */
/* random_image (synthetic.cpp:25-31), scene_image (:33-64), as float32. */
void fbf_random_image_f32(int width, int height, unsigned long long seed, float* out);
void fbf_scene_image_f32(int width, int height, unsigned long long seed, float* out);
/* BASELINE configs 0/1/3: n_sites Voronoi cells with U(0,255) values,
 * + N(0, noise^2), clipped to [0,255]. */
void fbf_voronoi_image_f32(int width, int height, int n_sites, double noise, unsigned long long seed,
                           int threads, float* out);
/* BASELINE configs 2/4: sum of 32 seeded 2-D sinusoids scaled to [0,255],
 * + n_sites Voronoi step edges (per-cell offset U(-64,64)), + N(0, noise^2),
 * clipped to [0,255]. */
void fbf_field_image_f32(int width, int height, int n_sites, double noise, unsigned long long seed,
                         int threads, float* out);

#ifdef __cplusplus
}
#endif

#endif /* FBF_H */
