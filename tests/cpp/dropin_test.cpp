// dropin_test.cpp -- the reference's own API, compiled against this repo's
// GPU drop-in headers (include/fastdeconv/{convolve,rl}.hpp shadow the
// reference's; image.hpp / psf.hpp are the reference's).  Mirrors the
// hot-path pins of /root/reference/proj/tests/test_convolve.cpp and
// test_rl.cpp with the fp32 tolerances of the B200 path; values are checked
// against the CPU oracle (oracle/liboracle.so, test infrastructure).
//
// usage: dropin_test [--cpu-only]     exit status = number of failed checks
//        dropin_test --time W H ITERS   wall time of rlDeconvolve(Image) through the drop-in
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "fastdeconv/rl.hpp"
#include "oracle.h"

using namespace fastdeconv;

static int g_fail = 0, g_pass = 0;

static void check(bool ok, const std::string& what) {
    std::printf("%s  %s\n", ok ? "PASS" : "FAIL", what.c_str());
    (ok ? g_pass : g_fail)++;
}

template <typename F>
static bool throws_with(F&& f, const char* needle) {
    try {
        f();
    } catch (const std::exception& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    }
    return false;
}

static Image randomImage(std::mt19937& rng, int w, int h, double lo = 0.0, double hi = 255.0) {
    std::uniform_real_distribution<double> d(lo, hi);
    Image img(w, h);
    for (double& v : img.data()) v = static_cast<float>(d(rng));  // fp32-representable inputs
    return img;
}

// oracle PSF from a reference Psf (normalised weights as the reference holds them)
static orc_psf* toOracle(const Psf& psf) {
    if (const auto* p = std::get_if<DensePsf>(&psf))
        return orc_psf_dense(p->width(), p->height(), p->anchorX(), p->anchorY(), p->weights().data());
    if (const auto* c = std::get_if<UniformConvexPsf>(&psf)) {
        std::vector<int> dy, lo, hi;
        for (const auto& r : c->rows()) {
            dy.push_back(r.dy);
            lo.push_back(r.xMin);
            hi.push_back(r.xMax);
        }
        return orc_psf_convex((int)dy.size(), dy.data(), lo.data(), hi.data());
    }
    const auto& s = std::get<SparsePsf>(psf);
    std::vector<int> dx, dy;
    std::vector<double> w;
    for (const PsfTap& t : s.taps()) {
        dx.push_back(t.dx);
        dy.push_back(t.dy);
        w.push_back(t.w);
    }
    return orc_psf_sparse((int)dx.size(), dx.data(), dy.data(), w.data());
}

static Image oracleConv(const Image& img, const Psf& psf, OperatorKind k) {
    orc_psf* p = toOracle(psf);
    Image out(img.width(), img.height());
    orc_convolve(img.data().data(), img.width(), img.height(), p, (int)k, out.data().data(), nullptr);
    orc_psf_free(p);
    return out;
}

static double relErr(const Image& a, const Image& ref) {
    double scale = 0.0, err = 0.0;
    for (size_t i = 0; i < a.pixelCount(); ++i) {
        scale = std::max(scale, std::abs(ref.data()[i]));
        err = std::max(err, std::abs(a.data()[i] - ref.data()[i]));
    }
    return scale > 0 ? err / scale : err;
}

static double maxRel(const Image& a, const Image& ref) {
    double m = 0.0;
    for (size_t i = 0; i < a.pixelCount(); ++i)
        m = std::max(m, std::abs(a.data()[i] - ref.data()[i]) / std::abs(ref.data()[i]));
    return m;
}

static bool identical(const Image& a, const Image& b) {
    return a.sameSize(b) && std::memcmp(a.data().data(), b.data().data(), a.pixelCount() * sizeof(double)) == 0;
}

static void hostChecks() {
    // dispatch, proj/tests/test_convolve.cpp:251-278
    check(dispatch(Psf(makeDiscPsf(9))) == OperatorKind::GenericBox, "dispatch disc -> generic-box");
    check(dispatch(Psf(makeLinePsf(17))) == OperatorKind::Box1dCumulated, "dispatch line -> box1d-cumul");
    check(dispatch(Psf(makeBoxPsf(9, 9))) == OperatorKind::Box2dCumulated, "dispatch box -> box2d-cumul");
    check(dispatch(Psf(makeDiagonalPsf(9))) == OperatorKind::List, "dispatch diagonal -> list");
    check(dispatch(Psf(DensePsf(3, 1, 1, 0, {1.0, 2.0, 1.0}))) == OperatorKind::Naive, "dispatch blob -> naive");
    check(dispatch(Psf(SparsePsf({{-1, 0, 1.0}, {0, 0, 1.0}, {1, 0, 1.0}}))) == OperatorKind::Box1dCumulated,
          "dispatch line-shaped sparse -> box1d-cumul");
    check(dispatch(Psf(makeDiscPsf(9)), OperatorKind::List) == OperatorKind::List, "explicit preference honoured");
    check(throws_with([] { dispatch(Psf(makeBoxPsf(3, 3)), OperatorKind::Box1dSliding); }, "box1d-sliding"),
          "incompatible preference names the operator");
    check(throws_with([] { dispatch(Psf(SparsePsf({{0, 0, 1.0}, {1, 0, 2.0}})), OperatorKind::GenericBox); },
                      "cannot handle"),
          "non-uniform sparse refuses generic-box");
    bool names = true;
    for (int k = 0; k <= 8; ++k) names &= operatorKindFromName(operatorName((OperatorKind)k)) == (OperatorKind)k;
    check(names && supportsMasking(OperatorKind::Naive) && !supportsMasking(OperatorKind::GenericBox),
          "operator names round-trip, masking capability");
    check(throws_with([] { operatorKindFromName("boxcar"); }, "unknown operator"), "unknown operator name throws");
    // validation (rl.hpp:71-84) happens before any device work
    Image bad(4, 4, 1.0);
    bad(1, 1) = -3.0;
    check(throws_with([&] { rlDeconvolve(bad, Psf(makeBoxPsf(1, 1))); }, "nonnegative"), "negative input rejected");
    bad(1, 1) = std::numeric_limits<double>::quiet_NaN();
    check(throws_with([&] { rlDeconvolve(bad, Psf(makeBoxPsf(1, 1))); }, "non-finite"), "NaN input rejected");
    RlConfig c0;
    c0.epsilonDiv = 0.0;
    check(throws_with([&] { rlDeconvolve(Image(4, 4, 1.0), Psf(makeBoxPsf(1, 1)), c0); }, "epsilonDiv"),
          "epsilonDiv <= 0 rejected");
    // validation in double before the fp32 conversion: a tiny negative
    // (rounds to -0.0f) is still "nonnegative"-rejected like the reference
    bad(1, 1) = -1e-46;
    check(throws_with([&] { rlDeconvolve(bad, Psf(makeBoxPsf(1, 1))); }, "nonnegative"),
          "tiny negative (fp32 -0.0) rejected as negative");
    bad(1, 1) = 1e39;
    check(throws_with([&] { rlDeconvolve(bad, Psf(makeBoxPsf(1, 1))); }, "fp32 range"),
          "value beyond the fp32 range refused with its own message");
    // ConvPlan construction is host-only (dispatch), like the reference's
    bool built = false;
    try {
        const ConvPlan p(Psf(makeDiscPsf(9)));
        built = p.kind() == OperatorKind::GenericBox;
    } catch (...) {
    }
    check(built, "ConvPlan constructs and resolves its operator without touching the device");
    RlConfig cg;
    cg.op = OperatorKind::GenericBox;
    check(throws_with([&] { rlDeconvolveSelective(Image(4, 4, 1.0), Psf(makeDiscPsf(3)), cg, 0.1); },
                      "masked evaluation"),
          "selective RL refuses generic-box");
}

static void deviceChecks() {
    std::mt19937 rng(33);
    // frozen vectors, proj/tests/test_convolve.cpp:60-78
    const Image row(5, 1, std::vector<double>{1, 2, 3, 4, 5});
    const double expected[] = {4.0 / 3.0, 2.0, 3.0, 4.0, 14.0 / 3.0};
    const Image s = box1dSlidingConvolve(row, 3), c = box1dCumulatedConvolve(row, 3);
    bool frozen = true;
    for (int x = 0; x < 5; ++x) frozen &= std::abs(s(x, 0) - expected[x]) < 1e-6 && std::abs(c(x, 0) - expected[x]) < 1e-6;
    check(frozen, "box1d frozen example [1..5], M=3");

    // fast operators agree with the (oracle) naive operator, test_convolve.cpp:80-117
    double worst = 0.0;
    int comparisons = 0;
    std::uniform_int_distribution<int> size(5, 40);
    for (int trial = 0; trial < 6; ++trial) {
        const Image img = randomImage(rng, size(rng), size(rng));
        for (int m : {1, 2, 3, 9, 17}) {
            const Psf line(makeLinePsf(m)), box(makeBoxPsf(m, m)), disc(makeDiscPsf(m)), diag(makeDiagonalPsf(m));
            const Image rl = oracleConv(img, line, OperatorKind::Naive);
            const Image rb = oracleConv(img, box, OperatorKind::Naive);
            const Image rd = oracleConv(img, disc, OperatorKind::Naive);
            const Image rg = oracleConv(img, diag, OperatorKind::Naive);
            for (OperatorKind k : {OperatorKind::Box1dSliding, OperatorKind::Box1dCumulated, OperatorKind::List,
                                   OperatorKind::Naive}) {
                worst = std::max(worst, relErr(convolve(img, line, k), rl));
                ++comparisons;
            }
            for (OperatorKind k : {OperatorKind::Box2dSliding, OperatorKind::Box2dCumulated, OperatorKind::GenericBox,
                                   OperatorKind::List}) {
                worst = std::max(worst, relErr(convolve(img, box, k), rb));
                ++comparisons;
            }
            worst = std::max(worst, relErr(genericBoxConvolve(img, makeDiscPsf(m)), rd));
            worst = std::max(worst, relErr(listConvolve(img, toSparse(makeDiscPsf(m))), rd));
            worst = std::max(worst, relErr(listConvolve(img, makeDiagonalPsf(m)), rg));
            worst = std::max(worst, relErr(genericBoxConvolve(img, *asUniformConvex(diag)), rg));
            comparisons += 4;
        }
    }
    check(worst < 2e-6, "fast operators vs oracle naive: " + std::to_string(comparisons) + " comparisons, max rel " +
                            std::to_string(worst));

    // identity / constants, test_convolve.cpp:38-58
    const Image img = randomImage(rng, 9, 6);
    check(identical(naiveConvolve(img, makeBoxPsf(1, 1)), img) && identical(box1dSlidingConvolve(img, 1), img) &&
              identical(genericBoxConvolve(img, makeDiscPsf(1)), img),
          "identity PSFs reproduce the input bit-exactly");
    const Image cst(13, 9, 50.0);
    check(relErr(box2dSlidingConvolve(cst, 5, 3), cst) < 1e-6 && relErr(genericBoxConvolve(cst, makeDiscPsf(9)), cst) < 1e-6 &&
              relErr(listConvolve(cst, makeDiagonalPsf(7)), cst) < 1e-6,
          "constant images map to the same constant");

    // masked semantics, test_convolve.cpp:207-249
    const Image im2 = randomImage(rng, 12, 9), fb = randomImage(rng, 12, 9);
    const Psf dense(toDense(makeDiscPsf(3))), sparse(makeDiagonalPsf(5));
    std::vector<std::uint8_t> ones(im2.pixelCount(), 1), zeros(im2.pixelCount(), 0), mask(im2.pixelCount());
    std::bernoulli_distribution coin(0.5);
    for (auto& m : mask) m = coin(rng);
    const Image full = listConvolve(im2, std::get<SparsePsf>(sparse));
    const Image part = maskedConvolve(im2, sparse, OperatorKind::List, mask, fb);
    bool exact = true;
    for (size_t i = 0; i < part.pixelCount(); ++i)
        exact &= part.data()[i] == (mask[i] ? full.data()[i] : static_cast<double>(static_cast<float>(fb.data()[i])));
    check(identical(maskedConvolve(im2, dense, OperatorKind::Naive, ones, fb), naiveConvolve(im2, std::get<DensePsf>(dense))) &&
              identical(maskedConvolve(im2, sparse, OperatorKind::Auto, ones, fb), full) && exact,
          "masked convolution: all-active == full, random mask exact");
    check(throws_with([&] { maskedConvolve(im2, dense, OperatorKind::GenericBox, ones, fb); },
                      "does not support masked evaluation"),
          "masked generic-box refuses");

    // cost counters, test_convolve.cpp:293-348
    const Image ci = randomImage(rng, 48, 32);
    ConvCounters c9, c18, cb, cn;
    listConvolve(ci, toSparse(makeLinePsf(9)), &c9);
    listConvolve(ci, toSparse(makeLinePsf(18)), &c18);
    box2dCumulatedConvolve(ci, 17, 17, &cb);
    naiveConvolve(ci, toDense(makeDiscPsf(9)), &cn);
    const uint64_t px = 48 * 32;
    check(c9.perPixelOps == 9 * px && c18.perPixelOps == 18 * px && cb.perPixelOps == 4 * px && cn.perPixelOps == 81 * px,
          "cost counters follow the reference model");

    // RL invariants, test_rl.cpp
    RlConfig cfg;
    cfg.iterations = 5;
    std::uniform_int_distribution<int> ints(0, 255);
    Image f(14, 10);
    for (double& v : f.data()) v = ints(rng);
    const RlResult r = rlDeconvolve(f, Psf(makeBoxPsf(1, 1)), cfg);
    check(identical(r.image, f) && r.trace.records.size() == 5, "identity PSF is a bit-exact RL fixed point");
    cfg.iterations = 20;
    const Image k100(16, 12, 100.0);
    check(relErr(rlDeconvolve(k100, Psf(makeDiscPsf(5)), cfg).image, k100) < 1e-5, "constant images stay constant");
    RlConfig cn2;
    cn2.iterations = 12;
    cn2.op = OperatorKind::Naive;
    Image g(40, 40);
    std::uniform_real_distribution<double> u01(0.2, 1.0);
    for (double& v : g.data()) v = static_cast<float>(u01(rng));
    const Image fb2 = convolve(g, Psf(toDense(makeDiscPsf(5))), OperatorKind::Naive);
    const RlResult std12 = rlDeconvolve(fb2, Psf(toDense(makeDiscPsf(5))), cn2);
    const RlResult sel12 = rlDeconvolveSelective(fb2, Psf(toDense(makeDiscPsf(5))), cn2, 0.0);
    check(identical(std12.image, sel12.image) && sel12.trace.omittedPercent() == 0.0,
          "selective RL with threshold 0 is bit-identical to standard RL");
    RlConfig c25;
    c25.iterations = 25;
    c25.op = OperatorKind::Naive;
    const RlResult inf = rlDeconvolveSelective(fb2, Psf(toDense(makeDiscPsf(3))), c25,
                                               std::numeric_limits<double>::infinity(), 10);
    check(std::abs(inf.trace.omittedPercent() - 88.0) < 1e-9 && inf.trace.records[1].inactiveFraction == 1.0,
          "infinite threshold reduces to the reactivation schedule (88% omitted)");

    // RL parity vs the oracle on a seeded scene (max-rel <= 1e-4)
    Image scene(96, 80);
    for (int y = 0; y < 80; ++y)
        for (int x = 0; x < 96; ++x) scene(x, y) = (x / 12 + y / 10) % 3 == 0 ? 0.9 : 0.2;
    for (const Psf& psf : {Psf(makeLinePsf(15)), Psf(makeDiscPsf(9)), Psf(makeBoxPsf(15, 15))}) {
        const Image fo = convolve(scene, psf);
        RlConfig c40;
        c40.iterations = 40;
        const RlResult gr = rlDeconvolve(fo, psf, c40);
        orc_psf* op = toOracle(psf);
        Image ref(96, 80);
        orc_rl_deconvolve(fo.data().data(), 96, 80, op, 40, (int)dispatch(psf), 1e-8, 1, ref.data().data(), nullptr,
                          nullptr, nullptr);
        orc_psf_free(op);
        check(maxRel(gr.image, ref) <= 1e-4, "RL parity vs oracle (" + std::string(operatorName(dispatch(psf))) +
                                                 "), max-rel " + std::to_string(maxRel(gr.image, ref)));
    }
    // rlStep / rlStepPlanned
    const ConvPlan fwd(Psf(makeBoxPsf(3, 3)), OperatorKind::Naive), adj(adjoint(Psf(makeBoxPsf(3, 3))), OperatorKind::Naive);
    const Image s1 = rlStep(fb2, fb2, Psf(makeBoxPsf(3, 3)), cn2);
    const Image s2 = detail::rlStepPlanned(fb2, fb2, fwd, adj, cn2);
    check(identical(s1, s2), "rlStepPlanned == rlStep");
    // rlStepPlanned honours the caller's adjoint plan: with an asymmetric
    // PSF and the FORWARD plan passed as "adjoint" the step is
    // u * (h (x) (f / (h (x) u))), not rlStep's u * (h* (x) ...)
    {
        const Psf ha(DensePsf(3, 1, 1, 0, {1.0, 2.0, 5.0}));
        const ConvPlan fa(ha, OperatorKind::Naive);
        const Image u0 = randomImage(rng, 40, 24, 1.0, 2.0), f0 = randomImage(rng, 40, 24, 1.0, 2.0);
        const Image sp = detail::rlStepPlanned(u0, f0, fa, fa, cn2);
        const Image st = rlStep(u0, f0, ha, cn2);
        const Image v = oracleConv(u0, ha, OperatorKind::Naive);
        Image q(40, 24);
        for (size_t i = 0; i < q.data().size(); ++i) q.data()[i] = f0.data()[i] / std::max(v.data()[i], 1e-8);
        const Image c = oracleConv(q, ha, OperatorKind::Naive);
        Image ex(40, 24);
        for (size_t i = 0; i < ex.data().size(); ++i) ex.data()[i] = std::max(c.data()[i] * u0.data()[i], 0.0);
        check(maxRel(sp, ex) <= 1e-5 && maxRel(st, ex) > 1e-3,
              "rlStepPlanned uses the caller's adjoint plan (max-rel " + std::to_string(maxRel(sp, ex)) + ")");
    }
    // one ConvPlan shared by several threads (each on its own context)
    {
        const ConvPlan shared(Psf(makeDiscPsf(9)));
        std::vector<Image> in, seq, par(6);
        for (int t = 0; t < 6; ++t) in.push_back(randomImage(rng, 300 + 16 * t, 200 + 8 * t));
        for (int t = 0; t < 6; ++t) seq.push_back(shared.apply(in[t]));
        std::vector<std::thread> th;
        for (int t = 0; t < 6; ++t)
            th.emplace_back([&, t] {
                for (int rep = 0; rep < 3; ++rep) par[t] = shared.apply(in[t]);
            });
        for (auto& x : th) x.join();
        bool same = true;
        for (int t = 0; t < 6; ++t) same &= identical(par[t], seq[t]);
        check(same, "one ConvPlan applied concurrently from 6 threads == sequential results");
    }
    // a plan built on a worker thread stays valid after that thread exits
    {
        std::unique_ptr<ConvPlan> p;
        std::thread([&] {
            p = std::make_unique<ConvPlan>(Psf(makeBoxPsf(5, 3)));
            (void)p->engine();  // device representation built on this thread's context
        }).join();
        const Image img = randomImage(rng, 64, 48);
        check(maxRel(p->apply(img), oracleConv(img, Psf(makeBoxPsf(5, 3)), p->kind())) <= 2e-6,
              "plan used after its creating thread exited");
    }
}

// --time W H ITERS: wall time of the reference-API call rlDeconvolve(const
// Image&, ...) (doubles in, doubles out, 15 x 15 box) through the drop-in
static int timeDropIn(int w, int h, int iters) {
    Image f(w, h, 0.5);
    std::mt19937 rng(4);
    std::uniform_real_distribution<double> d(0.2, 1.0);
    for (int y = 0; y < h; y += 7)
        for (int x = 0; x < w; ++x) f.row(y)[x] = d(rng);
    const Psf psf = makeBoxPsf(15, 15);
    RlConfig cfg;
    cfg.iterations = iters;
    cfg.op = OperatorKind::Box2dSliding;
    for (int rep = 0; rep < 4; ++rep) {
        const auto t0 = std::chrono::steady_clock::now();
        const RlResult r = rlDeconvolve(f, psf, cfg);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::printf("rlDeconvolve(Image %dx%d, box 15x15, %d iterations): %.1f ms per call, %.0f Mpx*it/s "
                    "(device %.1f ms; u[1][1] = %.6f)\n",
                    w, h, iters, ms, (double)w * h * iters / ms / 1e3, r.trace.totalSeconds() * 1e3,
                    r.image.row(1)[1]);
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 4 && std::string(argv[1]) == "--time")
        return timeDropIn(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]));
    const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu-only";
    hostChecks();
    if (!cpu_only) deviceChecks();
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
