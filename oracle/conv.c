/*
 * conv.c -- oracle restatement of the spatial convolution operators
 * (TEST INFRASTRUCTURE ONLY, see oracle.h).
 *
 * Reference: /root/reference/proj/include/fastdeconv/convolve.hpp.
 * Contract (convolve.hpp:17-21): out(x,y) = sum_taps w(dx,dy) *
 * in(clamp(x+dx), clamp(y+dy)) -- correlation with replicate continuation
 * (image.hpp:81-102).  Each operator reproduces the reference's sequence of
 * double operations per output value; loops over *independent* outputs are
 * reordered / threaded freely, which keeps every value bit-identical.
 */
#include "oracle.h"
#include "plan.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* one replicate-padded scan line: buf[i] = img(clamp(i - l), clamp(y)),
 * i in [0, w + l + r)  (PaddedImage::assign, image.hpp:94-100) */
static void pad_row(const double* img, int w, int h, int y, int l, int r, double* buf) {
    const double* src = img + (size_t)clampi(y, 0, h - 1) * w;
    for (int i = 0; i < l; ++i) buf[i] = src[0];
    memcpy(buf + l, src, (size_t)w * sizeof(double));
    for (int i = 0; i < r; ++i) buf[l + w + i] = src[w - 1];
}

/* ------------------------------------------------------------------ plans */

void plan_free(orc_plan* pl) {
    orc_psf_free(pl->rep);
    pl->rep = NULL;
}

/* ConvPlan ctor, convolve.hpp:652-676 */
int plan_init(orc_plan* pl, const orc_psf* psf, int preference) {
    memset(pl, 0, sizeof(*pl));
    const int kind = orc_dispatch(psf, preference);
    if (kind < 0) return ORC_EINVAL;
    pl->kind = kind;
    switch (kind) {
        case ORC_NAIVE:
        case ORC_FOURIER:
            pl->rep = orc_psf_to_dense(psf);
            break;
        case ORC_LIST:
            pl->rep = orc_psf_to_sparse(psf);
            break;
        case ORC_GENERIC_BOX:
            pl->rep = orc_psf_as_convex(psf);
            break;
        case ORC_BOX1D_SLIDING:
        case ORC_BOX1D_CUMUL:
            orc_psf_as_line(psf, &pl->len, &pl->min_dx, &pl->dy);
            return ORC_OK;
        case ORC_BOX2D_SLIDING:
        case ORC_BOX2D_CUMUL:
            orc_psf_as_rect(psf, &pl->mx, &pl->my, &pl->min_dx, &pl->min_dy);
            return ORC_OK;
    }
    return pl->rep ? ORC_OK : ORC_EINVAL;
}

/* ------------------------------------------------------------- operators */

/* naiveInto + denseWindowSum, convolve.hpp:89-98,126-145.  Per output the
 * accumulation is acc += w[iy*mw+ix] * p over iy, then ix (raster order). */
static void naive_row(const double* img, int w, int h, const orc_psf* d, int y, double* rows,
                      double* acc) {
    const int mw = d->width, mh = d->height, ax = d->anchor_x, ay = d->anchor_y;
    const int l = ax, r = mw - 1 - ax, pw = w + l + r;
    for (int x = 0; x < w; ++x) acc[x] = 0.0;
    for (int iy = 0; iy < mh; ++iy) {
        pad_row(img, w, h, y + iy - ay, l, r, rows);
        const double* wr = d->weights + (size_t)iy * mw;
        for (int ix = 0; ix < mw; ++ix) {
            const double wv = wr[ix];
            const double* p = rows + ix;
            for (int x = 0; x < w; ++x) acc[x] += wv * p[x];
        }
    }
    (void)pw;
}

static double naive_px(const double* img, int w, int h, const orc_psf* d, int x, int y) {
    const int mw = d->width, mh = d->height, ax = d->anchor_x, ay = d->anchor_y;
    double acc = 0.0;
    for (int iy = 0; iy < mh; ++iy) {
        const double* src = img + (size_t)clampi(y + iy - ay, 0, h - 1) * w;
        const double* wr = d->weights + (size_t)iy * mw;
        for (int ix = 0; ix < mw; ++ix) acc += wr[ix] * src[clampi(x + ix - ax, 0, w - 1)];
    }
    return acc;
}

/* listInto + ListKernel::eval, convolve.hpp:101-120,151-169: tap order */
static void list_row(const double* img, int w, int h, const orc_psf* s, int y, double* rowbuf,
                     double* acc) {
    for (int x = 0; x < w; ++x) acc[x] = 0.0;
    for (int k = 0; k < s->n_taps; ++k) {
        const double* src = img + (size_t)clampi(y + s->tap_dy[k], 0, h - 1) * w;
        const int dx = s->tap_dx[k];
        const double wv = s->tap_w[k];
        /* rowbuf[x] = src[clamp(x + dx)] */
        for (int x = 0; x < w; ++x) rowbuf[x] = src[clampi(x + dx, 0, w - 1)];
        for (int x = 0; x < w; ++x) acc[x] += wv * rowbuf[x];
    }
}

static double list_px(const double* img, int w, int h, const orc_psf* s, int x, int y) {
    double acc = 0.0;
    for (int k = 0; k < s->n_taps; ++k)
        acc += s->tap_w[k] *
               img[(size_t)clampi(y + s->tap_dy[k], 0, h - 1) * w + clampi(x + s->tap_dx[k], 0, w - 1)];
    return acc;
}

/* genericBoxInto, convolve.hpp:177-212: window sum rebuilt at x=0 per row,
 * then sum += (p[x+xMax] - p[x-1+xMin]) per span row. */
static void generic_row(const double* img, int w, int h, const orc_psf* c, int y, double* out) {
    const int n = c->n_rows;
    const double scale = c->uniform_w;
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        const double* p = img + (size_t)clampi(y + c->row_dy[i], 0, h - 1) * w;
        for (int dx = c->row_xmin[i]; dx <= c->row_xmax[i]; ++dx) sum += p[clampi(dx, 0, w - 1)];
    }
    out[0] = sum * scale;
    for (int x = 1; x < w; ++x) {
        for (int i = 0; i < n; ++i) {
            const double* p = img + (size_t)clampi(y + c->row_dy[i], 0, h - 1) * w;
            sum += p[clampi(x + c->row_xmax[i], 0, w - 1)] - p[clampi(x - 1 + c->row_xmin[i], 0, w - 1)];
        }
        out[x] = sum * scale;
    }
}

/* box1dSlidingInto, convolve.hpp:217-244 */
static void box1d_sliding_row(const double* img, int w, int h, int len, int min_dx, int dy, int y,
                              double* out) {
    const double* p = img + (size_t)clampi(y + dy, 0, h - 1) * w;
    const double scale = 1.0 / (double)len;
    double sum = 0.0;
    for (int k = 0; k < len; ++k) sum += p[clampi(min_dx + k, 0, w - 1)];
    out[0] = sum * scale;
    for (int x = 1; x < w; ++x) {
        sum += p[clampi(x + min_dx + len - 1, 0, w - 1)] - p[clampi(x - 1 + min_dx, 0, w - 1)];
        out[x] = sum * scale;
    }
}

/* box1dCumulatedInto, convolve.hpp:246-280 (prefix sums over the padded line) */
static void box1d_cumul_row(const double* img, int w, int h, int len, int min_dx, int dy, int y,
                            double* padbuf, double* sums, double* out) {
    const int l = min_dx < 0 ? -min_dx : 0;
    const int r = min_dx + len - 1 > 0 ? min_dx + len - 1 : 0;
    const int pw = w + l + r;
    const int ox = min_dx + l;
    const double scale = 1.0 / (double)len;
    pad_row(img, w, h, y + dy, l, r, padbuf);
    sums[0] = padbuf[0];
    for (int i = 1; i < pw; ++i) sums[i] = sums[i - 1] + padbuf[i];
    const double* hi = sums + ox + len - 1;
    if (ox == 0) {
        out[0] = hi[0] * scale;
        for (int x = 1; x < w; ++x) out[x] = (hi[x] - sums[x - 1]) * scale;
    } else {
        const double* lo = sums + ox - 1;
        for (int x = 0; x < w; ++x) out[x] = (hi[x] - lo[x]) * scale;
    }
}

/* box2dSlidingInto, convolve.hpp:288-342 */
static void box2d_sliding(const double* img, int w, int h, const orc_plan* pl, double* out) {
    const int mx = pl->mx, my = pl->my, min_dx = pl->min_dx, min_dy = pl->min_dy;
    const int t = min_dy < 0 ? -min_dy : 0;
    const int b = min_dy + my - 1 > 0 ? min_dy + my - 1 : 0;
    const int ph = h + t + b;
    const int oy = min_dy + t;
    const double scale = 1.0 / ((double)mx * (double)my);
    double* mid = (double*)malloc((size_t)w * ph * sizeof(double));
    /* horizontal pass over every padded row (row py is image row clamp(py-t)) */
#pragma omp parallel for schedule(static)
    for (int py = 0; py < ph; ++py) {
        const double* p = img + (size_t)clampi(py - t, 0, h - 1) * w;
        double* m = mid + (size_t)py * w;
        double sum = 0.0;
        for (int k = 0; k < mx; ++k) sum += p[clampi(min_dx + k, 0, w - 1)];
        m[0] = sum;
        for (int x = 1; x < w; ++x) {
            sum += p[clampi(x + min_dx + mx - 1, 0, w - 1)] - p[clampi(x - 1 + min_dx, 0, w - 1)];
            m[x] = sum;
        }
    }
    /* vertical running sums: independent per column, so thread over columns */
    const int CH = 256;
    const int nchunks = (w + CH - 1) / CH;
#pragma omp parallel for schedule(static)
    for (int c = 0; c < nchunks; ++c) {
        const int x0 = c * CH, x1 = x0 + CH < w ? x0 + CH : w;
        double col[256];
        for (int x = x0; x < x1; ++x) col[x - x0] = 0.0;
        for (int k = 0; k < my; ++k) {
            const double* m = mid + (size_t)(oy + k) * w;
            for (int x = x0; x < x1; ++x) col[x - x0] += m[x];
        }
        for (int x = x0; x < x1; ++x) out[x] = col[x - x0] * scale;
        for (int y = 1; y < h; ++y) {
            const double* enter = mid + (size_t)(y + oy + my - 1) * w;
            const double* leave = mid + (size_t)(y - 1 + oy) * w;
            double* dst = out + (size_t)y * w;
            for (int x = x0; x < x1; ++x) {
                col[x - x0] += enter[x] - leave[x];
                dst[x] = col[x - x0] * scale;
            }
        }
    }
    free(mid);
}

/* box2dCumulatedInto, convolve.hpp:346-388 (global summed-area table) */
static void box2d_cumul(const double* img, int w, int h, const orc_plan* pl, double* out) {
    const int mx = pl->mx, my = pl->my, min_dx = pl->min_dx, min_dy = pl->min_dy;
    const int l = min_dx < 0 ? -min_dx : 0, r = min_dx + mx - 1 > 0 ? min_dx + mx - 1 : 0;
    const int t = min_dy < 0 ? -min_dy : 0, b = min_dy + my - 1 > 0 ? min_dy + my - 1 : 0;
    const int pw = w + l + r, ph = h + t + b;
    const int ox = min_dx + l, oy = min_dy + t;
    const double scale = 1.0 / ((double)mx * (double)my);
    const size_t sw = (size_t)pw + 1;
    double* sat = (double*)malloc(sw * ((size_t)ph + 1) * sizeof(double));
    double* p = (double*)malloc((size_t)pw * sizeof(double));
    for (size_t i = 0; i < sw; ++i) sat[i] = 0.0;
    for (int py = 0; py < ph; ++py) {
        pad_row(img, w, h, py - t, l, r, p);
        const double* prev = sat + (size_t)py * sw;
        double* cur = sat + (size_t)(py + 1) * sw;
        cur[0] = 0.0;
        for (int px = 0; px < pw; ++px) cur[px + 1] = p[px] + prev[px + 1] + cur[px] - prev[px];
    }
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        const double* top = sat + (size_t)(y + oy) * sw;
        const double* bot = sat + (size_t)(y + oy + my) * sw;
        double* dst = out + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            const int c0 = x + ox, c1 = x + ox + mx;
            dst[x] = (bot[c1] - top[c1] - bot[c0] + top[c0]) * scale;
        }
    }
    free(p);
    free(sat);
}

/* Cyclic correlation (the Fourier operator's contract, convolve.hpp:394-418,
 * evaluated as a direct wrap-around sum instead of an FFT). */
static void cyclic_direct(const double* img, int w, int h, const orc_psf* d, double* out) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int iy = 0; iy < d->height; ++iy)
                for (int ix = 0; ix < d->width; ++ix) {
                    const double wv = d->weights[(size_t)iy * d->width + ix];
                    if (wv == 0.0) continue;
                    int sx = (x + ix - d->anchor_x) % w;
                    int sy = (y + iy - d->anchor_y) % h;
                    if (sx < 0) sx += w;
                    if (sy < 0) sy += h;
                    acc += wv * img[(size_t)sy * w + sx];
                }
            out[(size_t)y * w + x] = acc;
        }
}

static void add_counters(uint64_t* c, uint64_t px, uint64_t per, uint64_t setup) {
    if (!c) return;
    c[0] += px;
    c[1] += per;
    c[2] += setup;
}

/* ConvPlan::applyInto, convolve.hpp:680-715 */
int plan_apply(const orc_plan* pl, const double* img, int w, int h, double* out, uint64_t* counters) {
    const uint64_t nx = (uint64_t)w, ny = (uint64_t)h;
    switch (pl->kind) {
        case ORC_NAIVE: {
            const orc_psf* d = pl->rep;
#pragma omp parallel
            {
                double* rows = (double*)malloc((size_t)(w + d->width) * sizeof(double));
#pragma omp for schedule(static)
                for (int y = 0; y < h; ++y) naive_row(img, w, h, d, y, rows, out + (size_t)y * w);
                free(rows);
            }
            add_counters(counters, nx * ny, nx * ny * (uint64_t)d->width * d->height, 0);
            return ORC_OK;
        }
        case ORC_LIST: {
            const orc_psf* s = pl->rep;
#pragma omp parallel
            {
                double* rb = (double*)malloc((size_t)w * sizeof(double));
#pragma omp for schedule(static)
                for (int y = 0; y < h; ++y) list_row(img, w, h, s, y, rb, out + (size_t)y * w);
                free(rb);
            }
            add_counters(counters, nx * ny, nx * ny * (uint64_t)s->n_taps, 0);
            return ORC_OK;
        }
        case ORC_GENERIC_BOX: {
            const orc_psf* c = pl->rep;
#pragma omp parallel for schedule(static)
            for (int y = 0; y < h; ++y) generic_row(img, w, h, c, y, out + (size_t)y * w);
            add_counters(counters, nx * ny, (nx - 1) * 2 * (uint64_t)c->n_rows * ny,
                         (uint64_t)c->support * ny);
            return ORC_OK;
        }
        case ORC_BOX1D_SLIDING:
#pragma omp parallel for schedule(static)
            for (int y = 0; y < h; ++y)
                box1d_sliding_row(img, w, h, pl->len, pl->min_dx, pl->dy, y, out + (size_t)y * w);
            add_counters(counters, nx * ny, (nx - 1) * 2 * ny, (uint64_t)pl->len * ny);
            return ORC_OK;
        case ORC_BOX1D_CUMUL: {
            const int l = pl->min_dx < 0 ? -pl->min_dx : 0;
            const int r = pl->min_dx + pl->len - 1 > 0 ? pl->min_dx + pl->len - 1 : 0;
            const int pw = w + l + r;
#pragma omp parallel
            {
                double* pb = (double*)malloc((size_t)pw * sizeof(double));
                double* sb = (double*)malloc((size_t)pw * sizeof(double));
#pragma omp for schedule(static)
                for (int y = 0; y < h; ++y)
                    box1d_cumul_row(img, w, h, pl->len, pl->min_dx, pl->dy, y, pb, sb,
                                    out + (size_t)y * w);
                free(pb);
                free(sb);
            }
            add_counters(counters, nx * ny, nx * 2 * ny, (uint64_t)pw * ny);
            return ORC_OK;
        }
        case ORC_BOX2D_SLIDING: {
            box2d_sliding(img, w, h, pl, out);
            const int t = pl->min_dy < 0 ? -pl->min_dy : 0;
            const int b = pl->min_dy + pl->my - 1 > 0 ? pl->min_dy + pl->my - 1 : 0;
            const uint64_t ph = ny + t + b;
            add_counters(counters, nx * ny, ph * (nx - 1) * 2 + (ny - 1) * nx * 2,
                         ph * (uint64_t)pl->mx + nx * (uint64_t)pl->my);
            return ORC_OK;
        }
        case ORC_BOX2D_CUMUL: {
            box2d_cumul(img, w, h, pl, out);
            const int l = pl->min_dx < 0 ? -pl->min_dx : 0;
            const int r = pl->min_dx + pl->mx - 1 > 0 ? pl->min_dx + pl->mx - 1 : 0;
            const int t = pl->min_dy < 0 ? -pl->min_dy : 0;
            const int b = pl->min_dy + pl->my - 1 > 0 ? pl->min_dy + pl->my - 1 : 0;
            add_counters(counters, nx * ny, nx * ny * 4,
                         (uint64_t)(w + l + r) * (uint64_t)(h + t + b) * 3);
            return ORC_OK;
        }
        case ORC_FOURIER:
            cyclic_direct(img, w, h, pl->rep, out);
            return ORC_OK;
    }
    return ORC_EINVAL;
}

/* ConvPlan::applyMaskedInto, convolve.hpp:433-510 + checkMaskArgs :425-431.
 * Active pixels get the operator value (same arithmetic as the full pass),
 * inactive ones the fallback.  Rows with many active pixels are evaluated
 * with the vectorised full-row path, sparse ones pixel by pixel. */
int plan_apply_masked(const orc_plan* pl, const double* img, int w, int h, const uint8_t* active,
                      const double* fallback, double* out, uint64_t* counters) {
    if (pl->kind != ORC_NAIVE && pl->kind != ORC_LIST) return ORC_EINVAL;
    uint64_t visited = 0;
#pragma omp parallel reduction(+ : visited)
    {
        double* acc = (double*)malloc((size_t)w * sizeof(double));
        double* rows = (double*)malloc((size_t)(w + (pl->kind == ORC_NAIVE ? pl->rep->width : 0)) *
                                       sizeof(double));
#pragma omp for schedule(dynamic, 4)
        for (int y = 0; y < h; ++y) {
            const uint8_t* act = active + (size_t)y * w;
            const double* fb = fallback + (size_t)y * w;
            double* dst = out + (size_t)y * w;
            int n_act = 0;
            for (int x = 0; x < w; ++x) n_act += act[x] != 0;
            visited += (uint64_t)n_act;
            if (n_act * 4 > w) {
                if (pl->kind == ORC_NAIVE)
                    naive_row(img, w, h, pl->rep, y, rows, acc);
                else
                    list_row(img, w, h, pl->rep, y, rows, acc);
                for (int x = 0; x < w; ++x) dst[x] = act[x] ? acc[x] : fb[x];
            } else {
                for (int x = 0; x < w; ++x)
                    dst[x] = !act[x] ? fb[x]
                             : pl->kind == ORC_NAIVE ? naive_px(img, w, h, pl->rep, x, y)
                                                     : list_px(img, w, h, pl->rep, x, y);
            }
        }
        free(acc);
        free(rows);
    }
    if (counters) {
        counters[0] += visited;
        counters[1] += visited * (pl->kind == ORC_NAIVE
                                      ? (uint64_t)pl->rep->width * pl->rep->height
                                      : (uint64_t)pl->rep->n_taps);
    }
    return ORC_OK;
}

int orc_convolve(const double* img, int w, int h, const orc_psf* psf, int kind, double* out,
                 uint64_t* counters) {
    if (w < 1 || h < 1) return ORC_EINVAL;
    orc_plan pl;
    int st = plan_init(&pl, psf, kind);
    if (st != ORC_OK) return st;
    st = plan_apply(&pl, img, w, h, out, counters);
    plan_free(&pl);
    return st;
}

/* maskedConvolve, convolve.hpp:762-770 */
int orc_masked_convolve(const double* img, int w, int h, const orc_psf* psf, int kind,
                        const uint8_t* active, const double* fallback, double* out,
                        uint64_t* counters) {
    if (kind == ORC_AUTO) kind = psf->repr == ORC_PSF_SPARSE ? ORC_LIST : ORC_NAIVE;
    if (kind != ORC_NAIVE && kind != ORC_LIST) return ORC_EINVAL;
    orc_plan pl;
    int st = plan_init(&pl, psf, kind);
    if (st != ORC_OK) return st;
    st = plan_apply_masked(&pl, img, w, h, active, fallback, out, counters);
    plan_free(&pl);
    return st;
}

/* Row-major run walk, convolve.hpp:450-465 (active runs only). */
int64_t orc_mask_runs(const uint8_t* active, int w, int h, int32_t* runs, int64_t max_runs) {
    int64_t n = 0;
    for (int y = 0; y < h; ++y) {
        const uint8_t* act = active + (size_t)y * w;
        int x = 0;
        while (x < w) {
            int end = x + 1;
            if (act[x]) {
                while (end < w && act[end]) ++end;
                if (n < max_runs) {
                    runs[3 * n] = y;
                    runs[3 * n + 1] = x;
                    runs[3 * n + 2] = end - x;
                }
                ++n;
            } else {
                while (end < w && !act[end]) ++end;
            }
            x = end;
        }
    }
    return n;
}

int64_t orc_active_list(const uint8_t* active, int64_t n, int64_t* idx, int64_t max_idx) {
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (active[i]) {
            if (k < max_idx) idx[k] = i;
            ++k;
        }
    return k;
}
