/* plan.h -- oracle-internal ConvPlan restatement (TEST INFRASTRUCTURE ONLY). */
#ifndef FD_ORACLE_PLAN_H
#define FD_ORACLE_PLAN_H
#include "oracle.h"

/* ConvPlan, convolve.hpp:650-753: resolved kind + prepared representation */
typedef struct {
    int kind;
    orc_psf* rep;         /* dense (naive/fourier), sparse (list), convex (generic) */
    int len, min_dx, dy;  /* LineShape */
    int mx, my, min_dy;   /* RectShape (min_dx shared) */
} orc_plan;

int plan_init(orc_plan* pl, const orc_psf* psf, int preference);
void plan_free(orc_plan* pl);
int plan_apply(const orc_plan* pl, const double* img, int w, int h, double* out,
               uint64_t* counters);
int plan_apply_masked(const orc_plan* pl, const double* img, int w, int h, const uint8_t* active,
                      const double* fallback, double* out, uint64_t* counters);
#endif
