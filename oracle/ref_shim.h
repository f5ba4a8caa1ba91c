/*
 * ref_shim.h -- extern "C" face of the UNMODIFIED reference library
 * (/root/reference/proj/include/fastdeconv, header-only C++20), compiled by
 * oracle/Makefile into oracle/_ref/libfdref.so.  TEST / BASELINE
 * INFRASTRUCTURE ONLY: used to pin the oracle restatement, to generate the
 * golden fixtures, and as the CPU arm of bench.py (--impl reference).
 */
#ifndef FD_REF_SHIM_H
#define FD_REF_SHIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PSF as raw arrays; repr 0 = DensePsf, 1 = UniformConvexPsf, 2 = SparsePsf */
typedef struct {
    int repr;
    int width, height, anchor_x, anchor_y;
    const double* weights;
    int n_rows;
    const int *row_dy, *row_xmin, *row_xmax;
    int n_taps;
    const int *tap_dx, *tap_dy;
    const double* tap_w;
} fdref_psf;

const char* fdref_last_error(void);
int fdref_dispatch(const fdref_psf* psf, int preference);
/* normalised taps of toSparse(psf) in reference order; returns count */
int fdref_psf_taps(const fdref_psf* psf, int adjoint, int* dx, int* dy, double* w, int cap);
int fdref_convolve(const fdref_psf* psf, int kind, const double* img, int w, int h, double* out,
                   uint64_t* counters);
int fdref_masked_convolve(const fdref_psf* psf, int kind, const double* img, int w, int h,
                          const uint8_t* active, const double* fallback, double* out,
                          uint64_t* counters);
int fdref_rl_deconvolve(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                        const double* f, int w, int h, double* u_out, double* max_change,
                        double* seconds);
int fdref_rl_selective(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                       double threshold, int period, const double* f, int w, int h,
                       double* u_out, double* inactive, double* max_change);
/* restated rl.hpp:218-255 loop on the reference's own ConvPlan::applyMaskedInto
 * and detail::quotientInto, deactivation held off for k < thin_start */
int fdref_rl_selective_from(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                            double threshold, int period, int thin_start, const double* f, int w,
                            int h, double* u_out, double* inactive, double* max_change,
                            uint8_t* masks_out);
int fdref_rl_step(const fdref_psf* psf, int op, double eps, int clamp, const double* u,
                  const double* f, int w, int h, double* out);
/* CPU baseline: `threads` std::threads each run rlDeconvolve for `iterations`
 * on an independent strip of `strip_rows` rows of f (plus PSF halo).
 * Returns wall seconds of the slowest thread; *px_it = core pixels x iterations. */
double fdref_bench_strips(const fdref_psf* psf, int op, const double* f, int w, int h,
                          int iterations, int threads, int strip_rows, double* px_it);

#ifdef __cplusplus
}
#endif
#endif
