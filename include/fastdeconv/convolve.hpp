// fastdeconv/convolve.hpp -- B200 drop-in for the reference's convolution
// operators (/root/reference/proj/include/fastdeconv/convolve.hpp).
//
// Put this repo's include/ directory BEFORE the reference's on the include
// path: this header and fastdeconv/rl.hpp shadow the reference's hot-path
// headers, while fastdeconv/image.hpp and fastdeconv/psf.hpp (the data model)
// still come from the reference.  Same names, signatures and exception
// behaviour; every operator runs on the GPU through the C ABI of
// libfdgpu.so (include/fdgpu.h).  No CPU fallback: without a CUDA device the
// compute calls throw std::runtime_error.
//
// Numerics: the device computes in fp32 (the reference in fp64); results are
// fp32-rounded values widened to double.  ConvCounters are filled from the
// reference cost model (analytic), so counter-based checks see the same
// numbers as with the CPU operators.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <variant>
#include <vector>

#include "fastdeconv/image.hpp"
#include "fastdeconv/psf.hpp"
#include "fdgpu.h"

namespace fastdeconv {

/// Operator families of the reference (convolve.hpp:22-32); numbering is the
/// C ABI's fdg_op.
enum class OperatorKind {
    Naive = FDG_OP_NAIVE,
    List = FDG_OP_LIST,
    GenericBox = FDG_OP_GENERIC_BOX,
    Box2dSliding = FDG_OP_BOX2D_SLIDING,
    Box2dCumulated = FDG_OP_BOX2D_CUMUL,
    Box1dSliding = FDG_OP_BOX1D_SLIDING,
    Box1dCumulated = FDG_OP_BOX1D_CUMUL,
    Fourier = FDG_OP_FOURIER,
    Auto = FDG_OP_AUTO,
};

namespace gpu_detail {

inline constexpr std::string_view kNames[] = {"naive",         "list",        "generic-box",
                                              "box2d-sliding", "box2d-cumul", "box1d-sliding",
                                              "box1d-cumul",   "fourier",     "auto"};

[[noreturn]] inline void raise(int status) {
    const std::string msg = fdg_last_error();
    if (status == FDG_EINVAL) throw std::invalid_argument(msg);
    if (status == FDG_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

inline void check(int status) {
    if (status != FDG_OK) raise(status);
}

/// Per-thread device context on `device` (private stream, scratch and
/// pinned staging), created on first use: concurrent calls from different
/// threads share nothing (the reference API is pure and reentrant).
inline fdg_ctx* context(int device) {
    thread_local std::map<int, std::shared_ptr<fdg_ctx>> ctxs;
    std::shared_ptr<fdg_ctx>& ctx = ctxs[device];
    if (!ctx) {
        fdg_ctx* c = nullptr;
        check(fdg_ctx_create(device, &c));
        ctx = std::shared_ptr<fdg_ctx>(c, fdg_ctx_destroy);
    }
    return ctx.get();
}

/// ... on the calling thread's current CUDA device
inline fdg_ctx* context() {
    int device = 0;
    check(fdg_get_device(&device));
    return context(device);
}

/// rl.hpp:71-84's pixel checks on the caller's double values, before the
/// fp32 conversion of the GPU path (a tiny negative would round to -0.0 and
/// pass a check in fp32).  Finite values beyond the fp32 range cannot be
/// represented on the device: refused with their own message.
inline void validatePixels(const Image& f, const char* where) {
    for (double v : f.data()) {
        if (!std::isfinite(v)) throw std::invalid_argument(std::string(where) + ": input image has non-finite pixels");
        if (v < 0.0) throw std::invalid_argument(std::string(where) + ": input image must be nonnegative");
    }
    for (double v : f.data())
        if (v > static_cast<double>(FLT_MAX))
            throw std::invalid_argument(std::string(where) + ": input pixel exceeds the fp32 range of the GPU path");
}

/// fdg_psf_desc view of a reference Psf (owns the flattened arrays).
class Desc {
public:
    explicit Desc(const Psf& psf) {
        d_ = fdg_psf_desc{};
        if (const auto* p = std::get_if<DensePsf>(&psf)) {
            d_.repr = FDG_PSF_DENSE;
            d_.width = p->width();
            d_.height = p->height();
            d_.anchor_x = p->anchorX();
            d_.anchor_y = p->anchorY();
            d_.weights = p->weights().data();
        } else if (const auto* c = std::get_if<UniformConvexPsf>(&psf)) {
            d_.repr = FDG_PSF_UNIFORM_CONVEX;
            for (const auto& r : c->rows()) {
                dy_.push_back(r.dy);
                lo_.push_back(r.xMin);
                hi_.push_back(r.xMax);
            }
            d_.n_rows = static_cast<int>(dy_.size());
            d_.row_dy = dy_.data();
            d_.row_xmin = lo_.data();
            d_.row_xmax = hi_.data();
        } else {
            const auto& s = std::get<SparsePsf>(psf);
            d_.repr = FDG_PSF_SPARSE;
            for (const PsfTap& t : s.taps()) {
                dy_.push_back(t.dy);
                lo_.push_back(t.dx);
                w_.push_back(t.w);
            }
            d_.n_taps = static_cast<int>(w_.size());
            d_.tap_dx = lo_.data();
            d_.tap_dy = dy_.data();
            d_.tap_w = w_.data();
        }
    }
    const fdg_psf_desc* get() const { return &d_; }

private:
    fdg_psf_desc d_;
    std::vector<int> dy_, lo_, hi_;
    std::vector<double> w_;
};

/// [0, n) split over a few threads for the pixel-type conversions of large
/// images (the device works in fp32, Image holds doubles)
template <typename F>
inline void parallelRanges(std::size_t n, F&& body) {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned nt = n >= (std::size_t(1) << 22) ? std::min(16u, hw ? hw : 1u) : 1u;
    if (nt <= 1) {
        body(std::size_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back([&body, n, t, nt] { body(n * t / nt, n * (t + 1) / nt); });
    for (std::thread& x : th) x.join();
}

inline std::vector<float> toFloat(const Image& img) {
    const std::vector<double>& d = img.data();
    std::vector<float> out(d.size());
    parallelRanges(d.size(), [&](std::size_t a, std::size_t b) {
        for (std::size_t i = a; i < b; ++i) out[i] = static_cast<float>(d[i]);
    });
    return out;
}

inline Image fromFloat(const std::vector<float>& v, int w, int h) {
    std::vector<double> out(v.size());
    parallelRanges(v.size(), [&](std::size_t a, std::size_t b) {
        for (std::size_t i = a; i < b; ++i) out[i] = static_cast<double>(v[i]);
    });
    return Image(w, h, std::move(out));
}

}  // namespace gpu_detail

inline std::string_view operatorName(OperatorKind kind) {
    const int k = static_cast<int>(kind);
    return (k >= 0 && k <= 8) ? gpu_detail::kNames[k] : std::string_view("unknown");
}

inline OperatorKind operatorKindFromName(std::string_view name) {
    for (int k = 0; k <= 8; ++k)
        if (gpu_detail::kNames[k] == name) return static_cast<OperatorKind>(k);
    throw std::invalid_argument("unknown operator name: " + std::string(name));
}

/// Only the per-pixel operators evaluate masked (convolve.hpp:59-61).
inline bool supportsMasking(OperatorKind kind) {
    return kind == OperatorKind::Naive || kind == OperatorKind::List;
}

/// Reference cost-model counters (convolve.hpp:66-70).
struct ConvCounters {
    std::uint64_t pixels = 0;
    std::uint64_t perPixelOps = 0;
    std::uint64_t setupOps = 0;
};

/// Kept for signature compatibility; device buffers live in the GPU context.
struct ConvWorkspace {};

namespace detail {
inline void ensureSize(Image& out, int width, int height) {
    if (out.width() != width || out.height() != height) out = Image(width, height);
}
}  // namespace detail

inline bool operatorAcceptsPsf(OperatorKind kind, const Psf& psf) {
    int ok = 0;
    gpu_detail::check(fdg_operator_accepts(static_cast<int>(kind), gpu_detail::Desc(psf).get(), &ok));
    return ok != 0;
}

/// convolve.hpp:627-643 -- resolved by libfdgpu's plan logic (host only).
inline OperatorKind dispatch(const Psf& psf, OperatorKind preference = OperatorKind::Auto) {
    int kind = 0;
    gpu_detail::check(fdg_dispatch(gpu_detail::Desc(psf).get(), static_cast<int>(preference), &kind));
    return static_cast<OperatorKind>(kind);
}

/// A PSF bound to its resolved operator and its device-resident
/// representation (convolve.hpp:650-753).  Construction is host-only like the
/// reference's (dispatch); the device representation is built on first use
/// on the calling thread's current device and is immutable afterwards, so
/// copies and concurrent applications from several threads (each on its
/// own context) are safe.
class ConvPlan {
public:
    explicit ConvPlan(const Psf& psf, OperatorKind preference = OperatorKind::Auto)
        : kind_(dispatch(psf, preference)), psf_(psf), state_(std::make_shared<State>()) {}

    OperatorKind kind() const { return kind_; }
    /// the PSF the plan was built from
    const Psf& psf() const { return psf_; }

    /// the device plan (libfdgpu handle), built once
    fdg_plan* native() const {
        std::call_once(state_->once, [this] {
            fdg_plan* p = nullptr;
            gpu_detail::check(fdg_plan_create(gpu_detail::context(), gpu_detail::Desc(psf_).get(),
                                              static_cast<int>(kind_), &p));
            state_->plan = std::shared_ptr<fdg_plan>(p, fdg_plan_destroy);
        });
        return state_->plan.get();
    }

    /// the calling thread's context on the plan's device
    fdg_ctx* callerContext() const { return gpu_detail::context(fdg_plan_device(native())); }

    void applyInto(const Image& img, ConvWorkspace&, Image& out, ConvCounters* counters = nullptr) const {
        const int w = img.width(), h = img.height();
        const std::vector<float> in = gpu_detail::toFloat(img);
        std::vector<float> res(in.size());
        gpu_detail::check(fdg_conv_apply_ctx(callerContext(), native(), in.data(), w, h, res.data()));
        out = gpu_detail::fromFloat(res, w, h);
        addCounters(counters, w, h);
    }

    Image apply(const Image& img, ConvCounters* counters = nullptr) const {
        ConvWorkspace ws;
        Image out;
        applyInto(img, ws, out, counters);
        return out;
    }

    void applyMaskedInto(const Image& img, const std::vector<std::uint8_t>& active, const Image& fallback,
                         ConvWorkspace&, Image& out, ConvCounters* counters = nullptr) const {
        if (!supportsMasking(kind_)) throw std::invalid_argument("operator does not support masked evaluation");
        if (!img.sameSize(fallback))
            throw std::invalid_argument("maskedConvolve: fallback dimensions differ from input");
        if (active.size() != img.pixelCount())
            throw std::invalid_argument("maskedConvolve: mask size differs from input");
        const int w = img.width(), h = img.height();
        const std::vector<float> in = gpu_detail::toFloat(img), fb = gpu_detail::toFloat(fallback);
        std::vector<float> res(in.size());
        gpu_detail::check(fdg_conv_apply_masked_ctx(callerContext(), native(), in.data(), w, h, active.data(),
                                                    fb.data(), res.data()));
        out = gpu_detail::fromFloat(res, w, h);
        if (counters) {
            std::uint64_t c[3];
            gpu_detail::check(fdg_op_counters(gpu_detail::Desc(psf_).get(), static_cast<int>(kind_), w, h, c));
            std::uint64_t visited = 0;
            for (std::uint8_t a : active) visited += a != 0;
            const std::uint64_t n = static_cast<std::uint64_t>(w) * h;
            counters->pixels += visited;
            counters->perPixelOps += visited * (n ? c[1] / n : 0);
        }
    }

    Image applyMasked(const Image& img, const std::vector<std::uint8_t>& active, const Image& fallback,
                      ConvCounters* counters = nullptr) const {
        ConvWorkspace ws;
        Image out;
        applyMaskedInto(img, active, fallback, ws, out, counters);
        return out;
    }

    /// the device engine serving this plan ("box", "taps", "dense", ...)
    std::string engine() const { return fdg_plan_engine(native()); }

private:
    struct State {
        std::once_flag once;
        std::shared_ptr<fdg_plan> plan;
    };

    void addCounters(ConvCounters* counters, int w, int h) const {
        if (!counters) return;
        std::uint64_t c[3];
        gpu_detail::check(fdg_op_counters(gpu_detail::Desc(psf_).get(), static_cast<int>(kind_), w, h, c));
        counters->pixels += c[0];
        counters->perPixelOps += c[1];
        counters->setupOps += c[2];
    }

    OperatorKind kind_;
    Psf psf_;
    std::shared_ptr<State> state_;  // shared by copies: one device plan
};

inline Image convolve(const Image& img, const Psf& psf, OperatorKind kind = OperatorKind::Auto,
                      ConvCounters* counters = nullptr) {
    return ConvPlan(psf, kind).apply(img, counters);
}

/// Auto resolves within the maskable subset (convolve.hpp:762-770).
inline Image maskedConvolve(const Image& img, const Psf& psf, OperatorKind kind,
                            const std::vector<std::uint8_t>& active, const Image& fallback,
                            ConvCounters* counters = nullptr) {
    if (kind == OperatorKind::Auto)
        kind = std::holds_alternative<SparsePsf>(psf) ? OperatorKind::List : OperatorKind::Naive;
    if (!supportsMasking(kind)) throw std::invalid_argument("operator does not support masked evaluation");
    return ConvPlan(psf, kind).applyMasked(img, active, fallback, counters);
}

// ---- one-shot operators (convolve.hpp:517-601)
inline Image naiveConvolve(const Image& img, const DensePsf& psf, ConvCounters* c = nullptr) {
    return convolve(img, Psf(psf), OperatorKind::Naive, c);
}
inline Image listConvolve(const Image& img, const SparsePsf& psf, ConvCounters* c = nullptr) {
    return convolve(img, Psf(psf), OperatorKind::List, c);
}
inline Image genericBoxConvolve(const Image& img, const UniformConvexPsf& psf, ConvCounters* c = nullptr) {
    return convolve(img, Psf(psf), OperatorKind::GenericBox, c);
}
inline Image box1dSlidingConvolve(const Image& img, int length, ConvCounters* c = nullptr) {
    if (length < 1) throw std::invalid_argument("box1dSlidingConvolve: length must be >= 1");
    return convolve(img, Psf(makeLinePsf(length)), OperatorKind::Box1dSliding, c);
}
inline Image box1dCumulatedConvolve(const Image& img, int length, ConvCounters* c = nullptr) {
    if (length < 1) throw std::invalid_argument("box1dCumulatedConvolve: length must be >= 1");
    return convolve(img, Psf(makeLinePsf(length)), OperatorKind::Box1dCumulated, c);
}
inline Image box2dSlidingConvolve(const Image& img, int mx, int my, ConvCounters* c = nullptr) {
    if (mx < 1 || my < 1) throw std::invalid_argument("box2dSlidingConvolve: sizes must be >= 1");
    return convolve(img, Psf(makeBoxPsf(mx, my)), OperatorKind::Box2dSliding, c);
}
inline Image box2dCumulatedConvolve(const Image& img, int mx, int my, ConvCounters* c = nullptr) {
    if (mx < 1 || my < 1) throw std::invalid_argument("box2dCumulatedConvolve: sizes must be >= 1");
    return convolve(img, Psf(makeBoxPsf(mx, my)), OperatorKind::Box2dCumulated, c);
}
/// Cyclic (wrap-around) correlation -- the Fourier operator's contract,
/// evaluated directly on the device.
inline Image fourierConvolve(const Image& img, const DensePsf& psf) {
    return convolve(img, Psf(psf), OperatorKind::Fourier);
}
inline Image maskedNaiveConvolve(const Image& img, const DensePsf& psf, const std::vector<std::uint8_t>& active,
                                 const Image& fallback, ConvCounters* c = nullptr) {
    return maskedConvolve(img, Psf(psf), OperatorKind::Naive, active, fallback, c);
}
inline Image maskedListConvolve(const Image& img, const SparsePsf& psf, const std::vector<std::uint8_t>& active,
                                const Image& fallback, ConvCounters* c = nullptr) {
    return maskedConvolve(img, Psf(psf), OperatorKind::List, active, fallback, c);
}

}  // namespace fastdeconv
