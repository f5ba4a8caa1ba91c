/*
 * psf.c -- oracle restatement of the PSF model (TEST INFRASTRUCTURE ONLY,
 * see oracle.h).  Follows /root/reference/proj/include/fastdeconv/psf.hpp:
 * constructors + normalisation (:26-170), adjoint (:280-308), representation
 * conversions (:314-375) and shape classification (:399-464), plus the
 * operator acceptance / dispatch rules of convolve.hpp:607-643.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static orc_psf* psf_alloc(int repr) {
    orc_psf* p = (orc_psf*)calloc(1, sizeof(orc_psf));
    if (p) p->repr = repr;
    return p;
}

void orc_psf_free(orc_psf* p) {
    if (!p) return;
    free(p->weights);
    free(p->row_dy);
    free(p->row_xmin);
    free(p->row_xmax);
    free(p->tap_dx);
    free(p->tap_dy);
    free(p->tap_w);
    free(p);
}

/* DensePsf ctor, psf.hpp:30-46: validate, then divide by the raster-order sum */
orc_psf* orc_psf_dense(int w, int h, int ax, int ay, const double* weights) {
    if (w < 1 || h < 1) return NULL;
    if (ax < 0 || ax >= w || ay < 0 || ay >= h) return NULL;
    const size_t n = (size_t)w * h;
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double v = weights[i];
        if (!(v >= 0.0) || !isfinite(v)) return NULL;
        sum += v;
    }
    if (sum <= 0.0) return NULL;
    orc_psf* p = psf_alloc(ORC_PSF_DENSE);
    p->width = w;
    p->height = h;
    p->anchor_x = ax;
    p->anchor_y = ay;
    p->weights = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) p->weights[i] = weights[i] / sum;
    return p;
}

/* UniformConvexPsf ctor, psf.hpp:83-97 */
orc_psf* orc_psf_convex(int n, const int* dy, const int* xmin, const int* xmax) {
    if (n < 1) return NULL;
    long count = 0;
    for (int i = 0; i < n; ++i) {
        if (xmin[i] > xmax[i]) return NULL;
        if (i > 0 && dy[i] != dy[i - 1] + 1) return NULL;
        count += xmax[i] - xmin[i] + 1;
    }
    orc_psf* p = psf_alloc(ORC_PSF_CONVEX);
    p->n_rows = n;
    p->row_dy = (int*)malloc(n * sizeof(int));
    p->row_xmin = (int*)malloc(n * sizeof(int));
    p->row_xmax = (int*)malloc(n * sizeof(int));
    memcpy(p->row_dy, dy, n * sizeof(int));
    memcpy(p->row_xmin, xmin, n * sizeof(int));
    memcpy(p->row_xmax, xmax, n * sizeof(int));
    p->support = (int)count;
    p->uniform_w = 1.0 / (double)p->support;
    return p;
}

static int cmp_pair(const void* a, const void* b) {
    const int* x = (const int*)a;
    const int* y = (const int*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/* SparsePsf ctor, psf.hpp:126-142: positive weights, no duplicate offsets */
orc_psf* orc_psf_sparse(int n, const int* dx, const int* dy, const double* w) {
    if (n < 1) return NULL;
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        if (!(w[i] > 0.0) || !isfinite(w[i])) return NULL;
        sum += w[i];
    }
    int* keys = (int*)malloc(2 * (size_t)n * sizeof(int));
    for (int i = 0; i < n; ++i) {
        keys[2 * i] = dy[i];
        keys[2 * i + 1] = dx[i];
    }
    qsort(keys, n, 2 * sizeof(int), cmp_pair);
    for (int i = 1; i < n; ++i)
        if (keys[2 * i] == keys[2 * i - 2] && keys[2 * i + 1] == keys[2 * i - 1]) {
            free(keys);
            return NULL;
        }
    free(keys);
    orc_psf* p = psf_alloc(ORC_PSF_SPARSE);
    p->n_taps = n;
    p->tap_dx = (int*)malloc(n * sizeof(int));
    p->tap_dy = (int*)malloc(n * sizeof(int));
    p->tap_w = (double*)malloc(n * sizeof(double));
    for (int i = 0; i < n; ++i) {
        p->tap_dx[i] = dx[i];
        p->tap_dy[i] = dy[i];
        p->tap_w[i] = w[i] / sum;
    }
    return p;
}

orc_psf* orc_psf_copy(const orc_psf* p) {
    orc_psf* c = psf_alloc(p->repr);
    *c = *p;
    c->weights = NULL;
    c->row_dy = c->row_xmin = c->row_xmax = NULL;
    c->tap_dx = c->tap_dy = NULL;
    c->tap_w = NULL;
    if (p->weights) {
        size_t n = (size_t)p->width * p->height;
        c->weights = (double*)malloc(n * sizeof(double));
        memcpy(c->weights, p->weights, n * sizeof(double));
    }
    if (p->row_dy) {
        size_t n = (size_t)p->n_rows * sizeof(int);
        c->row_dy = (int*)malloc(n);
        c->row_xmin = (int*)malloc(n);
        c->row_xmax = (int*)malloc(n);
        memcpy(c->row_dy, p->row_dy, n);
        memcpy(c->row_xmin, p->row_xmin, n);
        memcpy(c->row_xmax, p->row_xmax, n);
    }
    if (p->tap_dx) {
        size_t n = (size_t)p->n_taps;
        c->tap_dx = (int*)malloc(n * sizeof(int));
        c->tap_dy = (int*)malloc(n * sizeof(int));
        c->tap_w = (double*)malloc(n * sizeof(double));
        memcpy(c->tap_dx, p->tap_dx, n * sizeof(int));
        memcpy(c->tap_dy, p->tap_dy, n * sizeof(int));
        memcpy(c->tap_w, p->tap_w, n * sizeof(double));
    }
    return c;
}

/* adjoint, psf.hpp:280-308: reflect about the origin.  The dense and sparse
 * results go through their constructors again (renormalisation included). */
orc_psf* orc_psf_adjoint(const orc_psf* p) {
    if (p->repr == ORC_PSF_DENSE) {
        const int w = p->width, h = p->height;
        double* rot = (double*)malloc((size_t)w * h * sizeof(double));
        for (int iy = 0; iy < h; ++iy)
            for (int ix = 0; ix < w; ++ix)
                rot[(size_t)(h - 1 - iy) * w + (w - 1 - ix)] = p->weights[(size_t)iy * w + ix];
        orc_psf* a = orc_psf_dense(w, h, w - 1 - p->anchor_x, h - 1 - p->anchor_y, rot);
        free(rot);
        return a;
    }
    if (p->repr == ORC_PSF_CONVEX) {
        const int n = p->n_rows;
        int* dy = (int*)malloc(n * sizeof(int));
        int* lo = (int*)malloc(n * sizeof(int));
        int* hi = (int*)malloc(n * sizeof(int));
        for (int i = 0; i < n; ++i) {
            const int s = n - 1 - i;
            dy[i] = -p->row_dy[s];
            lo[i] = -p->row_xmax[s];
            hi[i] = -p->row_xmin[s];
        }
        orc_psf* a = orc_psf_convex(n, dy, lo, hi);
        free(dy);
        free(lo);
        free(hi);
        return a;
    }
    const int n = p->n_taps;
    int* dx = (int*)malloc(n * sizeof(int));
    int* dy = (int*)malloc(n * sizeof(int));
    for (int i = 0; i < n; ++i) {
        dx[i] = -p->tap_dx[i];
        dy[i] = -p->tap_dy[i];
    }
    orc_psf* a = orc_psf_sparse(n, dx, dy, p->tap_w);
    free(dx);
    free(dy);
    return a;
}

/* toSparse, psf.hpp:314-332 */
orc_psf* orc_psf_to_sparse(const orc_psf* p) {
    if (p->repr == ORC_PSF_SPARSE) return orc_psf_copy(p);
    int cap = p->repr == ORC_PSF_DENSE ? p->width * p->height : p->support;
    int* dx = (int*)malloc(cap * sizeof(int));
    int* dy = (int*)malloc(cap * sizeof(int));
    double* w = (double*)malloc(cap * sizeof(double));
    int n = 0;
    if (p->repr == ORC_PSF_DENSE) {
        for (int iy = 0; iy < p->height; ++iy)
            for (int ix = 0; ix < p->width; ++ix) {
                const double v = p->weights[(size_t)iy * p->width + ix];
                if (v > 0.0) {
                    dx[n] = ix - p->anchor_x;
                    dy[n] = iy - p->anchor_y;
                    w[n] = v;
                    ++n;
                }
            }
    } else {
        for (int r = 0; r < p->n_rows; ++r)
            for (int x = p->row_xmin[r]; x <= p->row_xmax[r]; ++x) {
                dx[n] = x;
                dy[n] = p->row_dy[r];
                w[n] = p->uniform_w;
                ++n;
            }
    }
    orc_psf* s = orc_psf_sparse(n, dx, dy, w);
    free(dx);
    free(dy);
    free(w);
    return s;
}

/* toDense, psf.hpp:336-375 (denseFromTaps keeps the origin inside the grid) */
orc_psf* orc_psf_to_dense(const orc_psf* p) {
    if (p->repr == ORC_PSF_DENSE) return orc_psf_copy(p);
    orc_psf* s = orc_psf_to_sparse(p);
    if (!s) return NULL;
    int mnx = 0, mxx = 0, mny = 0, mxy = 0;
    for (int i = 0; i < s->n_taps; ++i) {
        if (s->tap_dx[i] < mnx) mnx = s->tap_dx[i];
        if (s->tap_dx[i] > mxx) mxx = s->tap_dx[i];
        if (s->tap_dy[i] < mny) mny = s->tap_dy[i];
        if (s->tap_dy[i] > mxy) mxy = s->tap_dy[i];
    }
    const int w = mxx - mnx + 1, h = mxy - mny + 1;
    double* grid = (double*)calloc((size_t)w * h, sizeof(double));
    for (int i = 0; i < s->n_taps; ++i)
        grid[(size_t)(s->tap_dy[i] - mny) * w + (s->tap_dx[i] - mnx)] += s->tap_w[i];
    orc_psf* d = orc_psf_dense(w, h, -mnx, -mny, grid);
    free(grid);
    orc_psf_free(s);
    return d;
}

/* detail::sortedTaps (psf.hpp:399-405): taps of toSparse sorted by (dy, dx).
 * Offsets are unique, so any correct sort gives the reference order. */
typedef struct {
    int dy, dx;
    double w;
} tap_t;

static int cmp_tap(const void* a, const void* b) {
    const tap_t* x = (const tap_t*)a;
    const tap_t* y = (const tap_t*)b;
    if (x->dy != y->dy) return x->dy < y->dy ? -1 : 1;
    if (x->dx != y->dx) return x->dx < y->dx ? -1 : 1;
    return 0;
}

static tap_t* sorted_taps(const orc_psf* p, int* n_out) {
    orc_psf* s = orc_psf_to_sparse(p);
    if (!s) {
        *n_out = 0;
        return NULL;
    }
    tap_t* t = (tap_t*)malloc(s->n_taps * sizeof(tap_t));
    for (int i = 0; i < s->n_taps; ++i) {
        t[i].dy = s->tap_dy[i];
        t[i].dx = s->tap_dx[i];
        t[i].w = s->tap_w[i];
    }
    qsort(t, s->n_taps, sizeof(tap_t), cmp_tap);
    *n_out = s->n_taps;
    orc_psf_free(s);
    return t;
}

/* detail::uniformWeights, psf.hpp:407-412 */
static int uniform_weights(const tap_t* t, int n) {
    const double expected = 1.0 / (double)n;
    for (int i = 0; i < n; ++i)
        if (fabs(t[i].w - expected) > 1e-12) return 0;
    return 1;
}

/* asUniformLine, psf.hpp:416-425 */
int orc_psf_as_line(const orc_psf* p, int* length, int* min_dx, int* dy) {
    int n;
    tap_t* t = sorted_taps(p, &n);
    int ok = t && uniform_weights(t, n);
    for (int i = 0; ok && i < n; ++i) {
        if (t[i].dy != t[0].dy) ok = 0;
        if (i > 0 && t[i].dx != t[i - 1].dx + 1) ok = 0;
    }
    if (ok) {
        *length = n;
        *min_dx = t[0].dx;
        *dy = t[0].dy;
    }
    free(t);
    return ok;
}

/* asUniformRect, psf.hpp:427-442 */
int orc_psf_as_rect(const orc_psf* p, int* mx, int* my, int* min_dx, int* min_dy) {
    int n;
    tap_t* t = sorted_taps(p, &n);
    int ok = t && uniform_weights(t, n);
    if (ok) {
        const int x0 = t[0].dx, y0 = t[0].dy, x1 = t[n - 1].dx, y1 = t[n - 1].dy;
        const long w = (long)x1 - x0 + 1, h = (long)y1 - y0 + 1;
        if (w * h != (long)n) ok = 0;
        int k = 0;
        for (int yy = y0; ok && yy <= y1; ++yy)
            for (int xx = x0; ok && xx <= x1; ++xx, ++k)
                if (t[k].dx != xx || t[k].dy != yy) ok = 0;
        if (ok) {
            *mx = (int)w;
            *my = (int)h;
            *min_dx = x0;
            *min_dy = y0;
        }
    }
    free(t);
    return ok;
}

/* asUniformConvex, psf.hpp:444-464 */
orc_psf* orc_psf_as_convex(const orc_psf* p) {
    if (p->repr == ORC_PSF_CONVEX) return orc_psf_copy(p);
    int n;
    tap_t* t = sorted_taps(p, &n);
    if (!t || !uniform_weights(t, n)) {
        free(t);
        return NULL;
    }
    int* dy = (int*)malloc(n * sizeof(int));
    int* lo = (int*)malloc(n * sizeof(int));
    int* hi = (int*)malloc(n * sizeof(int));
    int rows = 0, i = 0, ok = 1;
    while (ok && i < n) {
        const int row_dy = t[i].dy;
        const int x0 = t[i].dx;
        int x1 = x0;
        ++i;
        while (i < n && t[i].dy == row_dy) {
            if (t[i].dx != x1 + 1) {
                ok = 0;
                break;
            }
            x1 = t[i].dx;
            ++i;
        }
        if (!ok) break;
        if (rows > 0 && row_dy != dy[rows - 1] + 1) {
            ok = 0;
            break;
        }
        dy[rows] = row_dy;
        lo[rows] = x0;
        hi[rows] = x1;
        ++rows;
    }
    orc_psf* c = ok ? orc_psf_convex(rows, dy, lo, hi) : NULL;
    free(t);
    free(dy);
    free(lo);
    free(hi);
    return c;
}

/* operatorAcceptsPsf, convolve.hpp:607-625 */
int orc_operator_accepts(int kind, const orc_psf* p) {
    int a, b, c, d;
    switch (kind) {
        case ORC_NAIVE:
        case ORC_LIST:
        case ORC_FOURIER:
        case ORC_AUTO:
            return 1;
        case ORC_GENERIC_BOX: {
            orc_psf* cv = orc_psf_as_convex(p);
            int ok = cv != NULL;
            orc_psf_free(cv);
            return ok;
        }
        case ORC_BOX2D_SLIDING:
        case ORC_BOX2D_CUMUL:
            return orc_psf_as_rect(p, &a, &b, &c, &d);
        case ORC_BOX1D_SLIDING:
        case ORC_BOX1D_CUMUL:
            return orc_psf_as_line(p, &a, &b, &c);
    }
    return 0;
}

/* dispatch, convolve.hpp:627-643 */
int orc_dispatch(const orc_psf* p, int preference) {
    int a, b, c, d;
    if (preference == ORC_AUTO) {
        if (orc_psf_as_line(p, &a, &b, &c)) return ORC_BOX1D_CUMUL;
        if (orc_psf_as_rect(p, &a, &b, &c, &d)) return ORC_BOX2D_CUMUL;
        if (p->repr == ORC_PSF_CONVEX) return ORC_GENERIC_BOX;
        if (p->repr == ORC_PSF_SPARSE) return ORC_LIST;
        return ORC_NAIVE;
    }
    if (preference < 0 || preference > ORC_AUTO) return -1;
    return orc_operator_accepts(preference, p) ? preference : -1;
}
