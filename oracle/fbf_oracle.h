/*
 * fbf_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (double precision, single thread) restatement of the reference
 * fourierbf filtering path, used as the parity checker for the sm_100a
 * kernel. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product library never links it.
 *
 * Parity pin: tests/test_oracle.py checks every function here bit-for-bit
 * against the reference's own sources compiled verbatim into
 * oracle/_ref/libfbf_ref.so (see oracle/Makefile), and against the golden
 * fixtures under tests/golden/.
 */
#ifndef FBF_ORACLE_H
#define FBF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* BorderPolicy order follows image.hpp:38 {symmetric, replicate, zero}. */
enum { ORC_SYMMETRIC = 0, ORC_REPLICATE = 1, ORC_ZERO = 2 };
/* RangeKernelKind order follows kernels.hpp:8 {gaussian, exponential, cauchy}. */
enum { ORC_GAUSSIAN = 0, ORC_EXPONENTIAL = 1, ORC_CAUCHY = 2 };

int orc_map_border_index(int i, int n, int border);
/* taps must hold 2*ceil(3*theta)+1 doubles; returns the radius (or -1). */
int orc_spatial_radius(double theta);
int orc_build_spatial_kernel(double theta, double* taps);
/* values must hold 2R+1 doubles. */
int orc_sample_range_kernel(int kind, double sigma, int R, double* values);
double orc_frequency_of(int half_period);
double orc_evaluate_approximation(int K, int T, const double* coeffs, int t);
void orc_tabulate_approximation(int K, int T, int R, const double* coeffs, double* values);

/* Returns 0 on success, -1 invalid approximation, -2 pixel outside [0,R]. */
int orc_convolve_separable(const double* img, int w, int h, const double* taps, int radius,
                           int border, double* out);
int orc_fast_bilateral(const double* img, int w, int h, double theta, int K, int T, int R,
                       const double* coeffs, int border, double* out, long long* fallbacks);
int orc_brute_bilateral(const double* img, int w, int h, double theta, const double* range,
                        int R, int border, double* out, long long* fallbacks);

void orc_random_image(int w, int h, uint64_t seed, double* out);
void orc_scene_image(int w, int h, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif
