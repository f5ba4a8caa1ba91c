// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference
// library (see ref_shim.h).  Compiled only against
// /root/reference/proj/include; the output goes to oracle/_ref/ (git-ignored).
#include "ref_shim.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fastdeconv/rl.hpp"

using namespace fastdeconv;

namespace {

thread_local std::string g_err;

Psf makePsf(const fdref_psf* d) {
    if (d->repr == 0) {
        std::vector<double> w(d->weights, d->weights + (size_t)d->width * d->height);
        return DensePsf(d->width, d->height, d->anchor_x, d->anchor_y, std::move(w));
    }
    if (d->repr == 1) {
        std::vector<UniformConvexPsf::Row> rows;
        for (int i = 0; i < d->n_rows; ++i)
            rows.push_back({d->row_dy[i], d->row_xmin[i], d->row_xmax[i]});
        return UniformConvexPsf(std::move(rows));
    }
    std::vector<PsfTap> taps;
    for (int i = 0; i < d->n_taps; ++i) taps.push_back({d->tap_dx[i], d->tap_dy[i], d->tap_w[i]});
    return SparsePsf(std::move(taps));
}

Image makeImage(const double* p, int w, int h) {
    return Image(w, h, std::vector<double>(p, p + (size_t)w * h));
}

void copyOut(const Image& img, double* out) {
    std::memcpy(out, img.data().data(), img.pixelCount() * sizeof(double));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // namespace

extern "C" {

const char* fdref_last_error(void) { return g_err.c_str(); }

int fdref_dispatch(const fdref_psf* psf, int preference) {
    int out = -1;
    guarded([&] { out = (int)dispatch(makePsf(psf), (OperatorKind)preference); });
    return out;
}

int fdref_psf_taps(const fdref_psf* psf, int adj, int* dx, int* dy, double* w, int cap) {
    int n = -1;
    guarded([&] {
        Psf p = makePsf(psf);
        if (adj) p = adjoint(p);
        const std::vector<PsfTap> taps = psfTaps(p);
        n = (int)taps.size();
        for (int i = 0; i < n && i < cap; ++i) {
            dx[i] = taps[i].dx;
            dy[i] = taps[i].dy;
            w[i] = taps[i].w;
        }
    });
    return n;
}

int fdref_convolve(const fdref_psf* psf, int kind, const double* img, int w, int h, double* out,
                   uint64_t* counters) {
    return guarded([&] {
        ConvCounters c;
        const Image r = convolve(makeImage(img, w, h), makePsf(psf), (OperatorKind)kind, &c);
        copyOut(r, out);
        if (counters) {
            counters[0] = c.pixels;
            counters[1] = c.perPixelOps;
            counters[2] = c.setupOps;
        }
    });
}

int fdref_masked_convolve(const fdref_psf* psf, int kind, const double* img, int w, int h,
                          const uint8_t* active, const double* fallback, double* out,
                          uint64_t* counters) {
    return guarded([&] {
        ConvCounters c;
        std::vector<std::uint8_t> act(active, active + (size_t)w * h);
        const Image r = maskedConvolve(makeImage(img, w, h), makePsf(psf), (OperatorKind)kind, act,
                                       makeImage(fallback, w, h), &c);
        copyOut(r, out);
        if (counters) {
            counters[0] = c.pixels;
            counters[1] = c.perPixelOps;
            counters[2] = c.setupOps;
        }
    });
}

int fdref_rl_deconvolve(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                        const double* f, int w, int h, double* u_out, double* max_change,
                        double* seconds) {
    return guarded([&] {
        RlConfig cfg;
        cfg.iterations = iterations;
        cfg.op = (OperatorKind)op;
        cfg.epsilonDiv = eps;
        cfg.clampNonNegative = clamp != 0;
        const RlResult r = rlDeconvolve(makeImage(f, w, h), makePsf(psf), cfg);
        copyOut(r.image, u_out);
        for (size_t k = 0; k < r.trace.records.size(); ++k) {
            if (max_change) max_change[k] = r.trace.records[k].maxAbsChange;
            if (seconds) seconds[k] = r.trace.records[k].seconds;
        }
    });
}

int fdref_rl_selective(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                       double threshold, int period, const double* f, int w, int h,
                       double* u_out, double* inactive, double* max_change) {
    return guarded([&] {
        RlConfig cfg;
        cfg.iterations = iterations;
        cfg.op = (OperatorKind)op;
        cfg.epsilonDiv = eps;
        cfg.clampNonNegative = clamp != 0;
        const RlResult r =
            rlDeconvolveSelective(makeImage(f, w, h), makePsf(psf), cfg, threshold, period);
        copyOut(r.image, u_out);
        for (size_t k = 0; k < r.trace.records.size(); ++k) {
            if (inactive) inactive[k] = r.trace.records[k].inactiveFraction;
            if (max_change) max_change[k] = r.trace.records[k].maxAbsChange;
        }
    });
}

int fdref_rl_selective_from(const fdref_psf* psf, int iterations, int op, double eps, int clamp,
                            double threshold, int period, int thin_start, const double* f, int w,
                            int h, double* u_out, double* inactive, double* max_change,
                            uint8_t* masks_out) {
    return guarded([&] {
        const Psf hp = makePsf(psf);
        const Image fi = makeImage(f, w, h);
        OperatorKind kind = (OperatorKind)op;
        if (kind == OperatorKind::Auto)
            kind = std::holds_alternative<SparsePsf>(hp) ? OperatorKind::List : OperatorKind::Naive;
        const ConvPlan forward(hp, kind);
        const ConvPlan adjointPlan(adjoint(hp), kind);
        const std::size_t n = fi.pixelCount();
        Image u = fi;
        std::vector<std::uint8_t> act(n, 1);
        Image cachedV(w, h, 0.0), vNew(w, h), q, c;
        ConvWorkspace ws;
        for (int k = 0; k < iterations; ++k) {
            if (k % period == 0) std::fill(act.begin(), act.end(), std::uint8_t{1});
            std::size_t nin = 0;
            for (std::uint8_t a : act) nin += !a;
            if (masks_out) std::memcpy(masks_out + (size_t)k * n, act.data(), n);
            forward.applyMaskedInto(u, act, cachedV, ws, vNew);
            std::swap(cachedV, vNew);
            detail::quotientInto(fi, cachedV, eps, q);
            adjointPlan.applyMaskedInto(q, act, q, ws, c);
            double maxChange = 0.0;
            double* up = u.data().data();
            const double* cp = c.data().data();
            for (std::size_t i = 0; i < n; ++i) {
                if (!act[i]) continue;
                double value = cp[i] * up[i];
                if (clamp && value < 0.0) value = 0.0;
                const double d = std::abs(value - up[i]);
                if (d > maxChange) maxChange = d;
                if (k >= thin_start && d < threshold) act[i] = 0;
                up[i] = value;
            }
            if (inactive) inactive[k] = (double)nin / (double)n;
            if (max_change) max_change[k] = maxChange;
        }
        copyOut(u, u_out);
    });
}

int fdref_rl_step(const fdref_psf* psf, int op, double eps, int clamp, const double* u,
                  const double* f, int w, int h, double* out) {
    return guarded([&] {
        RlConfig cfg;
        cfg.op = (OperatorKind)op;
        cfg.epsilonDiv = eps;
        cfg.clampNonNegative = clamp != 0;
        copyOut(rlStep(makeImage(u, w, h), makeImage(f, w, h), makePsf(psf), cfg), out);
    });
}

double fdref_bench_strips(const fdref_psf* psf, int op, const double* f, int w, int h,
                          int iterations, int threads, int strip_rows, double* px_it) {
    const Psf hp = makePsf(psf);
    const SparsePsf s = toSparse(hp);
    const int top = std::max(0, -s.minDy()), bot = std::max(0, s.maxDy());
    std::vector<double> secs(threads, 0.0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int r0 = (int)(((long)t * strip_rows) % std::max(1, h - strip_rows + 1));
            const int a = std::max(0, r0 - top), b = std::min(h, r0 + strip_rows + bot);
            Image strip(w, b - a);
            std::memcpy(strip.data().data(), f + (size_t)a * w, (size_t)w * (b - a) * sizeof(double));
            RlConfig cfg;
            cfg.iterations = iterations;
            cfg.op = (OperatorKind)op;
            const auto t0 = std::chrono::steady_clock::now();
            const RlResult r = rlDeconvolve(strip, hp, cfg);
            const auto t1 = std::chrono::steady_clock::now();
            secs[t] = std::chrono::duration<double>(t1 - t0).count();
            (void)r;
        });
    }
    for (auto& th : pool) th.join();
    if (px_it) *px_it = (double)w * strip_rows * iterations * threads;
    return *std::max_element(secs.begin(), secs.end());
}

}  // extern "C"
