// examples/calibrate_gpu.cpp — the reference's calibrator, unchanged, driven
// by the GPU two-pass gradient.
//
// lanetape::gradient_descent (calibrate.hpp:127-219) only sees an
// Objective{value_and_grad, value} (calibrate.hpp:117-120). Here both
// callbacks are the B200 engine through lanetape_b200.hpp, under common
// random numbers, on synthetic targets manufactured at the truth
// (synthetic_targets, calibrate.hpp:224-227, evaluated on the GPU). The
// setting mirrors acceptance criterion 7 (tests/acceptance.cpp:337-394):
// kappa and theta start 50% off, all other parameters are frozen at the
// truth, and both must be recovered within 1%.
//
// Built by examples/Makefile against the reference headers in place; prints
// one JSON line. Usage: calibrate_gpu <model.json> [paths]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <span>

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.hpp"
#include "lanetape_b200_ref.hpp"

namespace lt = lanetape;
namespace gpu = lanetape_b200;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <model.json> [paths]\n", argv[0]);
        return 1;
    }
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const lt::ModelSpec spec = lt::load_model_spec(argv[1]);
        const std::vector<double> truth = lt::pack_params(spec.heston, spec.grid);
        gpu::Engine engine(gpu::to_gpu(spec));
        gpu::MCConfig cfg;
        cfg.paths = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : spec.mc.paths;
        cfg.seed = spec.mc.seed;
        const std::vector<double> targets = engine.estimate_means(truth, cfg).means;
        // a latency-bound loop of small calls: no timing events on the device
        // (ltg_set_timing), each call is its kernels alone
        engine.set_timing(false);

        const auto g = gpu::make_objective<lt::GradientReport>(engine, targets, cfg);
        // count the evaluations the calibrator makes (one gradient_of_G per
        // iteration, one estimate_means per Armijo trial, calibrate.hpp:149-217)
        std::size_t n_grad = 0, n_value = 0;
        lt::Objective objective{
            [&](std::span<const double> x) { ++n_grad; return g.value_and_grad(x); },
            [&](std::span<const double> x) { ++n_value; return g.value(x); }};

        lt::Bounds bounds{truth, truth};  // frozen at the truth except kappa, theta
        bounds.lo[0] = 1e-3;
        bounds.hi[0] = 25.0;
        bounds.lo[1] = 1e-5;
        bounds.hi[1] = 4.0;
        std::vector<double> x0(truth);
        x0[0] *= 1.5;
        x0[1] *= 1.5;
        lt::OptimizerConfig opt;
        opt.max_iters = 500;
        opt.g_rel_tol = 1e-10;
        opt.scales.resize(truth.size());
        for (std::size_t j = 0; j < truth.size(); ++j)
            opt.scales[j] = std::max(std::abs(truth[j]), 1e-2);

        const auto t1 = std::chrono::steady_clock::now();
        const lt::CalibrationResult res = lt::gradient_descent(objective, x0, bounds, opt);
        const auto t2 = std::chrono::steady_clock::now();
        const double sec = std::chrono::duration<double>(t2 - t0).count();
        const double cal = std::chrono::duration<double>(t2 - t1).count();
        const double G0 = res.trajectory.points.front().G;
        std::printf(
            "{\"converged\": %s, \"stop_reason\": \"%s\", \"iters\": %zu, \"G0\": %.17g, "
            "\"G\": %.17g, \"kappa\": %.17g, \"theta\": %.17g, \"kappa_err\": %.3e, "
            "\"theta_err\": %.3e, \"paths\": %zu, \"seconds\": %.3f, "
            "\"calibration_seconds\": %.4f, \"gradient_calls\": %zu, \"value_calls\": %zu, "
            "\"ms_per_evaluation\": %.4f}\n",
            res.converged ? "true" : "false", res.stop_reason.c_str(), res.iters, G0, res.G,
            res.params[0], res.params[1], std::fabs(res.params[0] - truth[0]) / truth[0],
            std::fabs(res.params[1] - truth[1]) / truth[1], cfg.paths, sec, cal, n_grad, n_value,
            1e3 * cal / double(std::max<std::size_t>(1, n_grad + n_value)));
        return 0;
    } catch (const gpu::EvalError& e) {
        std::fprintf(stderr, "numerical error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
