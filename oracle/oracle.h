/*
 * oracle.h -- CPU restatement of the fastdeconv Richardson-Lucy hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1304_7211_b200/,
 * include/) links, imports or calls this code.  It is the checker that the
 * CUDA path is compared against: tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py are its only users.
 *
 * Every function restates the reference algorithm in double precision with
 * the same operation order, so for naive / list / generic-box / box1d /
 * box2d / masked operators and both RL drivers its output is bit-identical
 * to /root/reference/proj/include/fastdeconv (pinned in tests/test_oracle.py
 * against oracle/_ref, the reference compiled from its own headers, and
 * against the reference's frozen test vectors in tests/golden/).
 *
 * Parallelism: OpenMP over output rows (columns for the box2d vertical pass).
 * Each output value is still produced by exactly the reference's sequence of
 * double operations, so the threaded oracle stays bit-identical.
 */
#ifndef FD_ORACLE_H
#define FD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* OperatorKind, same order as convolve.hpp:22-32 */
enum {
    ORC_NAIVE = 0,
    ORC_LIST = 1,
    ORC_GENERIC_BOX = 2,
    ORC_BOX2D_SLIDING = 3,
    ORC_BOX2D_CUMUL = 4,
    ORC_BOX1D_SLIDING = 5,
    ORC_BOX1D_CUMUL = 6,
    ORC_FOURIER = 7,
    ORC_AUTO = 8
};

/* Psf variant alternative, psf.hpp:173 */
enum { ORC_PSF_DENSE = 0, ORC_PSF_CONVEX = 1, ORC_PSF_SPARSE = 2 };

/* Status codes (exception classes of the reference). */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENAN = 2 };

typedef struct orc_psf {
    int repr;
    /* dense grid (psf.hpp:26-70) */
    int width, height, anchor_x, anchor_y;
    double* weights;
    /* uniform row-convex (psf.hpp:75-120) */
    int n_rows;
    int *row_dy, *row_xmin, *row_xmax;
    int support;
    double uniform_w;
    /* sparse taps (psf.hpp:124-170) */
    int n_taps;
    int *tap_dx, *tap_dy;
    double* tap_w;
} orc_psf;

/* constructors normalise exactly like the reference ctors; NULL on invalid */
orc_psf* orc_psf_dense(int w, int h, int ax, int ay, const double* weights);
orc_psf* orc_psf_convex(int n, const int* dy, const int* xmin, const int* xmax);
orc_psf* orc_psf_sparse(int n, const int* dx, const int* dy, const double* w);
void orc_psf_free(orc_psf* p);
orc_psf* orc_psf_copy(const orc_psf* p);
orc_psf* orc_psf_adjoint(const orc_psf* p);
orc_psf* orc_psf_to_sparse(const orc_psf* p);
orc_psf* orc_psf_to_dense(const orc_psf* p);
int orc_psf_as_line(const orc_psf* p, int* length, int* min_dx, int* dy);
int orc_psf_as_rect(const orc_psf* p, int* mx, int* my, int* min_dx, int* min_dy);
orc_psf* orc_psf_as_convex(const orc_psf* p);
int orc_operator_accepts(int kind, const orc_psf* p);
/* returns resolved kind, or -1 when the preference cannot handle the PSF */
int orc_dispatch(const orc_psf* p, int preference);

/* out = h (x) img with replicate continuation; counters may be NULL
 * (pixels, perPixelOps, setupOps).  Fourier is cyclic. */
int orc_convolve(const double* img, int w, int h, const orc_psf* psf, int kind, double* out,
                 uint64_t* counters);
int orc_masked_convolve(const double* img, int w, int h, const orc_psf* psf, int kind,
                        const uint8_t* active, const double* fallback, double* out,
                        uint64_t* counters);

/* rlDeconvolve (rl.hpp:140-179).  max_change/seconds: nullable, iterations
 * entries.  On NaN returns ORC_ENAN with *nan_iter set. */
int orc_rl_deconvolve(const double* f, int w, int h, const orc_psf* psf, int iterations, int op,
                      double eps, int clamp_nonneg, double* u_out, double* max_change,
                      double* seconds, int* nan_iter);

/* rlDeconvolveSelective (rl.hpp:187-257) with one extension: deactivation
 * (rl.hpp:245) is skipped for 0-based k < thin_start.
 * masks_out (nullable) receives the active mask each iteration's
 * convolutions used: iterations * w * h bytes. */
int orc_rl_selective(const double* f, int w, int h, const orc_psf* psf, int iterations, int op,
                     double eps, int clamp_nonneg, double threshold, int period, int thin_start,
                     double* u_out, double* inactive_frac, double* max_change,
                     uint8_t* masks_out, int* nan_iter);

/* one RL step (rl.hpp:101-137) */
int orc_rl_step(const double* u, const double* f, int w, int h, const orc_psf* psf, int op,
                double eps, int clamp_nonneg, double* u_out, double* max_change);

/* Row-major run walk of convolve.hpp:450-465: active runs (y, x0, len).
 * Returns the run count; writes at most max_runs triples. */
int64_t orc_mask_runs(const uint8_t* active, int w, int h, int32_t* runs, int64_t max_runs);
/* ordered active index list (row-major ascending) */
int64_t orc_active_list(const uint8_t* active, int64_t n, int64_t* idx, int64_t max_idx);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
