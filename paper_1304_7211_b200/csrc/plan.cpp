// plan.cpp -- host-side plan logic of libfdgpu: PSF validation, representation
// conversion, shape classification and operator dispatch.  Restates the
// reference rules so that "same API call -> same operator class" holds:
//   constructors / validation   psf.hpp:30-46, 83-97, 126-142
//   toSparse order               psf.hpp:314-332
//   adjoint (reflection)         psf.hpp:280-308
//   sortedTaps / uniformWeights  psf.hpp:399-412 (tolerance 1e-12)
//   asUniformLine/Rect/Convex    psf.hpp:416-464
//   operatorAcceptsPsf/dispatch  convolve.hpp:607-643
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>

#include "internal.h"

namespace fdg {

const char* op_name(int kind) {
    static const char* names[] = {"naive",         "list",          "generic-box",
                                  "box2d-sliding", "box2d-cumul",   "box1d-sliding",
                                  "box1d-cumul",   "fourier",       "auto"};
    return (kind >= 0 && kind <= 8) ? names[kind] : "unknown";
}

static bool fail(std::string* err, const char* msg) {
    if (err) *err = msg;
    return false;
}

bool psf_from_desc(const fdg_psf_desc* d, HostPsf* out, std::string* err) {
    if (!d) return fail(err, "null PSF descriptor");
    HostPsf p;
    p.repr = d->repr;
    if (d->repr == FDG_PSF_DENSE) {
        if (d->width < 1 || d->height < 1) return fail(err, "DensePsf: dimensions must be at least 1x1");
        if (d->anchor_x < 0 || d->anchor_x >= d->width || d->anchor_y < 0 || d->anchor_y >= d->height)
            return fail(err, "DensePsf: anchor must lie inside the grid");
        if (!d->weights) return fail(err, "DensePsf: weight count does not match dimensions");
        p.w = d->width;
        p.h = d->height;
        p.ax = d->anchor_x;
        p.ay = d->anchor_y;
        const size_t n = (size_t)p.w * p.h;
        double total = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double v = d->weights[i];
            if (!(v >= 0.0) || !std::isfinite(v))
                return fail(err, "DensePsf: weights must be finite and nonnegative");
            total += v;
        }
        if (total <= 0.0) return fail(err, "DensePsf: total weight must be positive");
        p.weights.resize(n);
        for (size_t i = 0; i < n; ++i) p.weights[i] = d->weights[i] / total;
    } else if (d->repr == FDG_PSF_UNIFORM_CONVEX) {
        if (d->n_rows < 1) return fail(err, "UniformConvexPsf: at least one support row required");
        for (int i = 0; i < d->n_rows; ++i) {
            const Span s{d->row_dy[i], d->row_xmin[i], d->row_xmax[i]};
            if (s.xmin > s.xmax) return fail(err, "UniformConvexPsf: row interval is empty");
            if (i > 0 && s.dy != p.rows.back().dy + 1)
                return fail(err, "UniformConvexPsf: row offsets must be contiguous and increasing");
            p.rows.push_back(s);
        }
    } else if (d->repr == FDG_PSF_SPARSE) {
        if (d->n_taps < 1) return fail(err, "SparsePsf: at least one tap required");
        double total = 0.0;
        std::set<std::pair<int, int>> seen;
        for (int i = 0; i < d->n_taps; ++i) {
            const double v = d->tap_w[i];
            if (!(v > 0.0) || !std::isfinite(v))
                return fail(err, "SparsePsf: weights must be finite and positive");
            if (!seen.insert({d->tap_dy[i], d->tap_dx[i]}).second)
                return fail(err, "SparsePsf: duplicate tap coordinates");
            total += v;
        }
        for (int i = 0; i < d->n_taps; ++i) p.taps.push_back({d->tap_dx[i], d->tap_dy[i], d->tap_w[i] / total});
    } else {
        return fail(err, "unknown PSF representation");
    }
    *out = std::move(p);
    return true;
}

static int support_count(const HostPsf& p) {
    int n = 0;
    for (const Span& s : p.rows) n += s.xmax - s.xmin + 1;
    return n;
}

std::vector<Tap> psf_taps(const HostPsf& p) {
    std::vector<Tap> t;
    if (p.repr == FDG_PSF_DENSE) {
        for (int iy = 0; iy < p.h; ++iy)
            for (int ix = 0; ix < p.w; ++ix) {
                const double v = p.weights[(size_t)iy * p.w + ix];
                if (v > 0.0) t.push_back({ix - p.ax, iy - p.ay, v});
            }
    } else if (p.repr == FDG_PSF_UNIFORM_CONVEX) {
        const double u = 1.0 / (double)support_count(p);
        for (const Span& s : p.rows)
            for (int dx = s.xmin; dx <= s.xmax; ++dx) t.push_back({dx, s.dy, u});
    } else {
        t = p.taps;
    }
    return t;
}

HostPsf psf_adjoint(const HostPsf& p) {
    HostPsf a;
    a.repr = p.repr;
    if (p.repr == FDG_PSF_DENSE) {
        a.w = p.w;
        a.h = p.h;
        a.ax = p.w - 1 - p.ax;
        a.ay = p.h - 1 - p.ay;
        a.weights.resize(p.weights.size());
        for (int iy = 0; iy < p.h; ++iy)
            for (int ix = 0; ix < p.w; ++ix)
                a.weights[(size_t)(p.h - 1 - iy) * p.w + (p.w - 1 - ix)] = p.weights[(size_t)iy * p.w + ix];
    } else if (p.repr == FDG_PSF_UNIFORM_CONVEX) {
        for (auto it = p.rows.rbegin(); it != p.rows.rend(); ++it) a.rows.push_back({-it->dy, -it->xmax, -it->xmin});
    } else {
        for (const Tap& t : p.taps) a.taps.push_back({-t.dx, -t.dy, t.w});
    }
    return a;
}

static std::vector<Tap> sorted(const HostPsf& p) {
    std::vector<Tap> t = psf_taps(p);
    std::sort(t.begin(), t.end(), [](const Tap& a, const Tap& b) { return a.dy != b.dy ? a.dy < b.dy : a.dx < b.dx; });
    return t;
}

static bool uniform(const std::vector<Tap>& t) {
    const double expect = 1.0 / (double)t.size();
    for (const Tap& x : t)
        if (std::fabs(x.w - expect) > 1e-12) return false;
    return true;
}

bool psf_as_line(const HostPsf& p, LineShape* out) {
    const std::vector<Tap> t = sorted(p);
    if (t.empty() || !uniform(t)) return false;
    for (size_t i = 0; i < t.size(); ++i) {
        if (t[i].dy != t[0].dy) return false;
        if (i && t[i].dx != t[i - 1].dx + 1) return false;
    }
    if (out) *out = {(int)t.size(), t[0].dx, t[0].dy};
    return true;
}

bool psf_as_rect(const HostPsf& p, RectShape* out) {
    const std::vector<Tap> t = sorted(p);
    if (t.empty() || !uniform(t)) return false;
    const int x0 = t.front().dx, y0 = t.front().dy, x1 = t.back().dx, y1 = t.back().dy;
    const long mx = (long)x1 - x0 + 1, my = (long)y1 - y0 + 1;
    if (mx * my != (long)t.size()) return false;
    size_t k = 0;
    for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x, ++k)
            if (t[k].dx != x || t[k].dy != y) return false;
    if (out) *out = {(int)mx, (int)my, x0, y0};
    return true;
}

bool psf_as_convex(const HostPsf& p, std::vector<Span>* out) {
    if (p.repr == FDG_PSF_UNIFORM_CONVEX) {
        if (out) *out = p.rows;
        return true;
    }
    const std::vector<Tap> t = sorted(p);
    if (t.empty() || !uniform(t)) return false;
    std::vector<Span> rows;
    for (size_t i = 0; i < t.size();) {
        Span s{t[i].dy, t[i].dx, t[i].dx};
        for (++i; i < t.size() && t[i].dy == s.dy; ++i) {
            if (t[i].dx != s.xmax + 1) return false;  // gap inside a row
            s.xmax = t[i].dx;
        }
        if (!rows.empty() && s.dy != rows.back().dy + 1) return false;  // gap between rows
        rows.push_back(s);
    }
    if (out) *out = rows;
    return true;
}

bool psf_accepts(int kind, const HostPsf& p) {
    switch (kind) {
        case FDG_OP_NAIVE:
        case FDG_OP_LIST:
        case FDG_OP_FOURIER:
        case FDG_OP_AUTO:
            return true;
        case FDG_OP_GENERIC_BOX:
            return psf_as_convex(p, nullptr);
        case FDG_OP_BOX2D_SLIDING:
        case FDG_OP_BOX2D_CUMUL:
            return psf_as_rect(p, nullptr);
        case FDG_OP_BOX1D_SLIDING:
        case FDG_OP_BOX1D_CUMUL:
            return psf_as_line(p, nullptr);
    }
    return false;
}

int psf_dispatch(const HostPsf& p, int preference, std::string* err) {
    if (preference == FDG_OP_AUTO) {
        if (psf_as_line(p, nullptr)) return FDG_OP_BOX1D_CUMUL;
        if (psf_as_rect(p, nullptr)) return FDG_OP_BOX2D_CUMUL;
        if (p.repr == FDG_PSF_UNIFORM_CONVEX) return FDG_OP_GENERIC_BOX;
        if (p.repr == FDG_PSF_SPARSE) return FDG_OP_LIST;
        return FDG_OP_NAIVE;
    }
    if (preference < 0 || preference > FDG_OP_AUTO) {
        if (err) *err = "unknown operator kind";
        return -1;
    }
    if (!psf_accepts(preference, p)) {
        if (err) {
            const char* kind = p.repr == FDG_PSF_DENSE ? "dense" : p.repr == FDG_PSF_UNIFORM_CONVEX ? "uniform-convex" : "sparse";
            char buf[160];
            std::snprintf(buf, sizeof buf, "operator '%s' cannot handle this %s PSF", op_name(preference), kind);
            *err = buf;
        }
        return -1;
    }
    return preference;
}

}  // namespace fdg
