// fastdeconv/rl.hpp -- B200 drop-in for the reference's Richardson-Lucy
// drivers (/root/reference/proj/include/fastdeconv/rl.hpp).
//
// Same types, signatures and exceptions; the whole iteration loop runs in
// libfdgpu (include/fdgpu.h) with u, f and the ratio image resident in HBM
// and the RL elementwise steps fused into the convolution epilogues.  The
// trace carries the per-iteration {iteration, inactiveFraction,
// maxAbsChange, seconds} (seconds from CUDA events on the device).
// Extension: rlDeconvolveSelective takes an optional thinStart (deactivation
// held off for 0-based iterations k < thinStart; 0 = the reference).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastdeconv/convolve.hpp"
#include "fastdeconv/image.hpp"
#include "fastdeconv/psf.hpp"

namespace fastdeconv {

/// rl.hpp:18-23
struct RlConfig {
    int iterations = 100;
    OperatorKind op = OperatorKind::Auto;
    double epsilonDiv = 1e-8;
    bool clampNonNegative = true;
};

struct RlIterationRecord {
    int iteration = 0;
    double inactiveFraction = 0;
    double maxAbsChange = 0;
    double seconds = 0;
};

struct RlTrace {
    std::vector<RlIterationRecord> records;

    double omittedPercent() const {
        if (records.empty()) return 0.0;
        double sum = 0.0;
        for (const RlIterationRecord& r : records) sum += r.inactiveFraction;
        return 100.0 * sum / static_cast<double>(records.size());
    }

    double totalSeconds() const {
        double sum = 0.0;
        for (const RlIterationRecord& r : records) sum += r.seconds;
        return sum;
    }
};

struct RlResult {
    Image image;
    RlTrace trace;
};

struct ActivityMask {
    std::vector<std::uint8_t> active;
    Image cachedV;
    double threshold = 0.0;
    int reactivationPeriod = 10;
};

enum class BoundaryMode { Cyclic, Replicate };

namespace gpu_detail {

inline fdg_rl_config toC(const RlConfig& cfg) {
    return fdg_rl_config{cfg.iterations, static_cast<int>(cfg.op), cfg.epsilonDiv, cfg.clampNonNegative ? 1 : 0};
}

inline RlTrace toTrace(const std::vector<fdg_rl_record>& recs) {
    RlTrace t;
    t.records.reserve(recs.size());
    for (const fdg_rl_record& r : recs)
        t.records.push_back({r.iteration, r.inactive_fraction, r.max_abs_change, r.seconds});
    return t;
}

/// the context handle, or NULL when no device exists (argument validation
/// still runs in the library; compute then reports the missing device)
inline fdg_ctx* contextOrNull() { return fdg_device_available() ? context() : nullptr; }

/// rl.hpp:71-84 in the reference's order (config, then pixels in double)
/// n doubles for a result the library fills completely.  std::vector<double>(n)
/// zero-fills single-threaded, faulting in every page on the way: 0.7 s for a
/// 16384^2 image against 0.12 s for the whole deconvolution.  With libstdc++
/// the storage is reserved and claimed without touching it (double is an
/// implicit-lifetime type: the library's writes are its initialisation), so
/// the pages are first touched by the library's parallel conversion pass;
/// elsewhere (or under the sanitizer's container annotations) the plain
/// zero-filled vector is returned.
inline std::vector<double> resultStorage(std::size_t n) {
#if defined(__GLIBCXX__) && !defined(_GLIBCXX_SANITIZE_VECTOR) && !defined(_GLIBCXX_DEBUG)
    struct Claim : std::vector<double> {
        explicit Claim(std::size_t count) {
            this->reserve(count);
            this->_M_impl._M_finish = this->_M_impl._M_start + count;
        }
    };
    Claim c(n);
    return std::vector<double>(std::move(static_cast<std::vector<double>&>(c)));
#else
    return std::vector<double>(n);
#endif
}

inline void validateRlConfig(const Image& f, const RlConfig& cfg, const char* where) {
    if (f.empty()) throw std::invalid_argument(std::string(where) + ": empty input image");
    if (cfg.iterations < 0) throw std::invalid_argument(std::string(where) + ": iterations must be >= 0");
    if (!(cfg.epsilonDiv > 0.0)) throw std::invalid_argument(std::string(where) + ": epsilonDiv must be positive");
}

inline void validateRlInputs(const Image& f, const RlConfig& cfg, const char* where) {
    validateRlConfig(f, cfg, where);
    validatePixels(f, where);
}

}  // namespace gpu_detail


/// rl.hpp:131-137
inline Image rlStep(const Image& u, const Image& f, const Psf& h, const RlConfig& cfg = {}) {
    if (!u.sameSize(f)) throw std::invalid_argument("rlStep: image dimensions differ");
    const std::vector<float> uf = gpu_detail::toFloat(u), ff = gpu_detail::toFloat(f);
    std::vector<float> out(uf.size());
    const fdg_rl_config c = gpu_detail::toC(cfg);
    double mc = 0.0;
    gpu_detail::check(fdg_rl_step(gpu_detail::contextOrNull(), gpu_detail::Desc(h).get(), &c, uf.data(), ff.data(),
                                  u.width(), u.height(), out.data(), &mc));
    return gpu_detail::fromFloat(out, u.width(), u.height());
}

/// rl.hpp:140-179
inline RlResult rlDeconvolve(const Image& f, const Psf& h, const RlConfig& cfg = {}) {
    // config checks here (rl.hpp:71-77), the pixel checks of rl.hpp:78-83 on
    // the doubles inside the library, in the pass that converts them
    gpu_detail::validateRlConfig(f, cfg, "rlDeconvolve");
    std::vector<double> u = gpu_detail::resultStorage(f.pixelCount());
    std::vector<fdg_rl_record> recs(static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 0));
    const fdg_rl_config c = gpu_detail::toC(cfg);
    gpu_detail::check(fdg_rl_deconvolve_f64(gpu_detail::contextOrNull(), gpu_detail::Desc(h).get(), &c,
                                            f.data().data(), f.width(), f.height(), u.data(),
                                            recs.empty() ? nullptr : recs.data()));
    return RlResult{Image(f.width(), f.height(), std::move(u)), gpu_detail::toTrace(recs)};
}

/// rl.hpp:187-257 (+ thinStart, see the header comment)
inline RlResult rlDeconvolveSelective(const Image& f, const Psf& h, const RlConfig& cfg, double threshold,
                                      int period = 10, int thinStart = 0) {
    gpu_detail::validateRlInputs(f, cfg, "rlDeconvolveSelective");
    const std::vector<float> ff = gpu_detail::toFloat(f);
    std::vector<float> u(ff.size());
    std::vector<fdg_rl_record> recs(static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 0));
    const fdg_rl_config c = gpu_detail::toC(cfg);
    gpu_detail::check(fdg_rl_deconvolve_selective(gpu_detail::contextOrNull(), gpu_detail::Desc(h).get(), &c, threshold,
                                                  period, thinStart, nullptr, nullptr, ff.data(), f.width(),
                                                  f.height(), u.data(), recs.empty() ? nullptr : recs.data()));
    return RlResult{gpu_detail::fromFloat(u, f.width(), f.height()), gpu_detail::toTrace(recs)};
}

/// rl.hpp:261-265: cyclic = the Fourier operator's wrap-around contract.
inline Image blurImage(const Image& g, const Psf& h, BoundaryMode mode) {
    if (mode == BoundaryMode::Cyclic) return fourierConvolve(g, toDense(h));
    return convolve(g, h, OperatorKind::Auto);
}

namespace detail {
/// rlStepPlanned (rl.hpp:101-125): one step with the caller's forward and
/// adjoint plans (their device representations, applied on the calling
/// thread's context).
inline Image rlStepPlanned(const Image& u, const Image& f, const ConvPlan& forward, const ConvPlan& adjointPlan,
                           const RlConfig& cfg, double* maxAbsChange = nullptr) {
    const std::vector<float> uf = gpu_detail::toFloat(u), ff = gpu_detail::toFloat(f);
    std::vector<float> out(uf.size());
    const fdg_rl_config cc = gpu_detail::toC(cfg);
    double mc = 0.0;
    gpu_detail::check(fdg_rl_step_planned(forward.callerContext(), forward.native(), adjointPlan.native(), &cc,
                                          uf.data(), ff.data(), u.width(), u.height(), out.data(), &mc));
    if (maxAbsChange) *maxAbsChange = mc;
    return gpu_detail::fromFloat(out, u.width(), u.height());
}
}  // namespace detail

}  // namespace fastdeconv
