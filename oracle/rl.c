/*
 * rl.c -- oracle restatement of the Richardson-Lucy drivers
 * (TEST INFRASTRUCTURE ONLY, see oracle.h).
 * Reference: /root/reference/proj/include/fastdeconv/rl.hpp.
 */
#include "oracle.h"
#include "plan.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* detail::validateRlInputs, rl.hpp:71-84 */
static int validate(const double* f, int w, int h, int iterations, double eps) {
    if (w < 1 || h < 1) return ORC_EINVAL;
    if (iterations < 0) return ORC_EINVAL;
    if (!(eps > 0.0)) return ORC_EINVAL;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        if (!isfinite(f[i])) return ORC_EINVAL;
        if (f[i] < 0.0) return ORC_EINVAL;
    }
    return ORC_OK;
}

/* detail::quotientInto, rl.hpp:86-94: q = f / std::max(v, eps) */
static void quotient(const double* f, const double* v, double eps, double* q, size_t n) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < (long)n; ++i) q[i] = f[i] / (v[i] < eps ? eps : v[i]);
}

/* forward = ConvPlan(h, op); adjoint = ConvPlan(adjoint(h), forward.kind())
 * (rl.hpp:142-143) */
static int make_plans(const orc_psf* psf, int op, orc_plan* fwd, orc_plan* adj) {
    int st = plan_init(fwd, psf, op);
    if (st != ORC_OK) return st;
    orc_psf* a = orc_psf_adjoint(psf);
    st = a ? plan_init(adj, a, fwd->kind) : ORC_EINVAL;
    orc_psf_free(a);
    if (st != ORC_OK) plan_free(fwd);
    return st;
}

/* rlDeconvolve, rl.hpp:140-179 */
int orc_rl_deconvolve(const double* f, int w, int h, const orc_psf* psf, int iterations, int op,
                      double eps, int clamp_nonneg, double* u_out, double* max_change,
                      double* seconds, int* nan_iter) {
    int st = validate(f, w, h, iterations, eps);
    if (st != ORC_OK) return st;
    orc_plan fwd, adj;
    st = make_plans(psf, op, &fwd, &adj);
    if (st != ORC_OK) return st;
    const size_t n = (size_t)w * h;
    double* u = u_out;
    memcpy(u, f, n * sizeof(double));
    double* v = (double*)malloc(n * sizeof(double));
    double* q = (double*)malloc(n * sizeof(double));
    double* c = (double*)malloc(n * sizeof(double));
    for (int k = 1; k <= iterations; ++k) {
        const double t0 = now_s();
        plan_apply(&fwd, u, w, h, v, NULL);
        quotient(f, v, eps, q, n);
        plan_apply(&adj, q, w, h, c, NULL);
        double max_d = 0.0;
        int any_nan = 0;
        /* update loop rl.hpp:164-171 (u is overwritten in place: each value
         * depends only on the same pixel, exactly like next/swap) */
#pragma omp parallel for schedule(static) reduction(max : max_d) reduction(| : any_nan)
        for (long i = 0; i < (long)n; ++i) {
            double value = c[i] * u[i];
            if (clamp_nonneg && value < 0.0) value = 0.0;
            const double d = fabs(value - u[i]);
            if (d > max_d) max_d = d;
            if (isnan(value)) any_nan = 1;
            u[i] = value;
        }
        const double t1 = now_s();
        if (any_nan) {
            if (nan_iter) *nan_iter = k;
            st = ORC_ENAN;
            break;
        }
        if (max_change) max_change[k - 1] = max_d;
        if (seconds) seconds[k - 1] = t1 - t0;
    }
    free(v);
    free(q);
    free(c);
    plan_free(&fwd);
    plan_free(&adj);
    return st;
}

/* rlStep / rlStepPlanned, rl.hpp:101-137 */
int orc_rl_step(const double* u, const double* f, int w, int h, const orc_psf* psf, int op,
                double eps, int clamp_nonneg, double* u_out, double* max_change) {
    orc_plan fwd, adj;
    int st = make_plans(psf, op, &fwd, &adj);
    if (st != ORC_OK) return st;
    const size_t n = (size_t)w * h;
    double* v = (double*)malloc(n * sizeof(double));
    double* q = (double*)malloc(n * sizeof(double));
    double* c = (double*)malloc(n * sizeof(double));
    plan_apply(&fwd, u, w, h, v, NULL);
    quotient(f, v, eps, q, n);
    plan_apply(&adj, q, w, h, c, NULL);
    double max_d = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double value = c[i] * u[i];
        if (clamp_nonneg && value < 0.0) value = 0.0;
        u_out[i] = value;
        const double d = fabs(value - u[i]);
        if (d > max_d) max_d = d;
    }
    if (max_change) *max_change = max_d;
    free(v);
    free(q);
    free(c);
    plan_free(&fwd);
    plan_free(&adj);
    return ORC_OK;
}

/* rlDeconvolveSelective, rl.hpp:187-257, with deactivation held off for
 * 0-based k < thin_start (thin_start = 0 is the reference). */
int orc_rl_selective(const double* f, int w, int h, const orc_psf* psf, int iterations, int op,
                     double eps, int clamp_nonneg, double threshold, int period, int thin_start,
                     double* u_out, double* inactive_frac, double* max_change,
                     uint8_t* masks_out, int* nan_iter) {
    int st = validate(f, w, h, iterations, eps);
    if (st != ORC_OK) return st;
    if (threshold < 0.0) return ORC_EINVAL;
    if (period < 1) return ORC_EINVAL;
    int kind = op;
    if (kind == ORC_AUTO) kind = psf->repr == ORC_PSF_SPARSE ? ORC_LIST : ORC_NAIVE;
    if (kind != ORC_NAIVE && kind != ORC_LIST) return ORC_EINVAL;
    orc_plan fwd, adj;
    st = plan_init(&fwd, psf, kind);
    if (st != ORC_OK) return st;
    orc_psf* a = orc_psf_adjoint(psf);
    st = plan_init(&adj, a, kind);
    orc_psf_free(a);
    if (st != ORC_OK) {
        plan_free(&fwd);
        return st;
    }
    const size_t n = (size_t)w * h;
    double* u = u_out;
    memcpy(u, f, n * sizeof(double));
    uint8_t* act = (uint8_t*)malloc(n);
    memset(act, 1, n);
    double* cached = (double*)calloc(n, sizeof(double));
    double* vnew = (double*)malloc(n * sizeof(double));
    double* q = (double*)malloc(n * sizeof(double));
    double* c = (double*)malloc(n * sizeof(double));
    for (int k = 0; k < iterations; ++k) {
        if (k % period == 0) memset(act, 1, n);
        size_t inactive = 0;
        for (size_t i = 0; i < n; ++i) inactive += !act[i];
        if (masks_out) memcpy(masks_out + (size_t)k * n, act, n);
        plan_apply_masked(&fwd, u, w, h, act, cached, vnew, NULL);
        double* tmp = cached;
        cached = vnew;
        vnew = tmp;
        quotient(f, cached, eps, q, n);
        plan_apply_masked(&adj, q, w, h, act, q, c, NULL);
        double max_d = 0.0;
        int any_nan = 0;
        const int may_thin = k >= thin_start;
#pragma omp parallel for schedule(static) reduction(max : max_d) reduction(| : any_nan)
        for (long i = 0; i < (long)n; ++i) {
            if (!act[i]) continue;
            double value = c[i] * u[i];
            if (clamp_nonneg && value < 0.0) value = 0.0;
            const double d = fabs(value - u[i]);
            if (d > max_d) max_d = d;
            if (may_thin && d < threshold) act[i] = 0;
            if (isnan(value)) any_nan = 1;
            u[i] = value;
        }
        if (any_nan) {
            if (nan_iter) *nan_iter = k + 1;
            st = ORC_ENAN;
            break;
        }
        if (inactive_frac) inactive_frac[k] = (double)inactive / (double)n;
        if (max_change) max_change[k] = max_d;
    }
    free(act);
    free(cached);
    free(vnew);
    free(q);
    free(c);
    plan_free(&fwd);
    plan_free(&adj);
    return st;
}
