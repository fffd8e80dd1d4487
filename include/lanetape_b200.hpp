// lanetape_b200.hpp — C++ host API over the C ABI (lanetape_b200.h).
//
// Mirrors the reference's calling surface for the ∇G path
// (/root/reference/proj/include/lanetape/):
//   ModelSpec / HestonParams / LeverageGrid / Instrument   heston.hpp:20-114
//   MCConfig, GradientReport, MeansResult                  expectation.hpp:25-82
//   gradient_of_G, estimate_means, finite_diff_gradient_of_G
//                                                          expectation.hpp:274-400
//   Objective {value_and_grad, value}                      calibrate.hpp:117-120
// Errors are raised like the reference's: std::invalid_argument (LTG_EINVAL),
// lanetape_b200::EvalError (LTG_ENUMERIC), std::runtime_error (LTG_ECUDA).
//
// The reference programs against a recorded Tape; the GPU engine is built
// from the model description the tape is recorded from
// (record_heston_program(ModelSpec), heston.hpp:327-329), so an Engine is the
// GPU counterpart of "record the program, freeze a Kernel".
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lanetape_b200.h"

namespace lanetape_b200 {

struct HestonParams {
    double mu = 0.0, kappa = 1.0, theta = 0.04, xi = 0.5, rho = -0.7, v0 = 0.04, s0 = 100.0;
};
struct LeverageGrid {
    std::vector<double> t_nodes, s_nodes, values;  // values t-major
};
struct Instrument {
    enum class Kind { Call, Put };
    Kind kind = Kind::Call;
    double strike = 100.0;
    std::size_t maturity_step = 1;
};
struct McSettings {
    std::size_t paths = 0, steps = 0;
    double dt = 0.0;
    std::uint64_t seed = 0;
};
struct ModelSpec {
    HestonParams heston;
    LeverageGrid grid;
    std::vector<Instrument> instruments;
    McSettings mc;
};

enum class MemoryMode { Recompute, Store };
enum class Precision { FP64, FP32 };

struct MCConfig {
    std::size_t paths = 0;
    std::uint64_t seed = 0;
    bool antithetic = false;
    int lane_width = 4;       // CPU knob, ignored by the GPU engine
    int worker_threads = 1;   // CPU knob, ignored by the GPU engine
    MemoryMode memory_mode = MemoryMode::Recompute;
    bool fresh_step2_paths = false;
    std::size_t store_limit_bytes = std::size_t{3} << 30;  // CPU knob
    Precision precision = Precision::FP64;
};

struct MeansResult {
    std::vector<double> means, std_errors;
    std::size_t paths = 0;
};

struct GradientReport {
    double G = 0.0;
    std::vector<double> means, lambda, grad;
    std::size_t paths = 0;
    std::string mode;
    std::uint64_t seed = 0;
};

// Draws fixed by the caller (rng.hpp:140-167 BufferDrawSource; a SampleSpace,
// expectation.hpp:46-54, is the same rows with paths = scenarios): row p holds
// the num_randoms() draws of path p.
struct BufferDraws {
    std::span<const double> draws;  // rows * dimension, path-major
    std::size_t dimension = 0;
};

struct SampleSpace {
    std::size_t scenarios = 0;
    std::size_t num_randoms = 0;
    std::vector<double> draws;  // scenario-major, scenarios * num_randoms
};

class EvalError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline std::vector<double> pack_params(const HestonParams& p, const LeverageGrid& g) {
    std::vector<double> x{p.kappa, p.theta, p.xi, p.rho, p.v0};
    x.insert(x.end(), g.values.begin(), g.values.end());
    return x;
}

namespace detail {
inline void check(int rc, const char* msg) {
    if (rc == LTG_OK) return;
    const std::string m = msg ? msg : "lanetape_b200 error";
    if (rc == LTG_EINVAL) throw std::invalid_argument(m);
    if (rc == LTG_ENUMERIC) throw EvalError(m);
    throw std::runtime_error(m);
}
inline ltg_mc_config to_c(const MCConfig& c) {
    ltg_mc_config o{};
    o.paths = c.paths;
    o.seed = c.seed;
    o.antithetic = c.antithetic ? 1 : 0;
    o.fresh_step2_paths = c.fresh_step2_paths ? 1 : 0;
    o.memory_mode = c.memory_mode == MemoryMode::Store ? LTG_MODE_STORE : LTG_MODE_RECOMPUTE;
    o.precision = c.precision == Precision::FP32 ? LTG_FP32 : LTG_FP64;
    return o;
}
}  // namespace detail

// A Heston-SLV program bound to one GPU, or (the devices constructor) to
// several GPUs of this process: every call then shards the paths over them
// (ltg_create_heston_devices) with the same results.
class Engine {
public:
    explicit Engine(const ModelSpec& s, int device = 0) : Engine(s, std::vector<int>{device}, false) {}
    Engine(const ModelSpec& s, const std::vector<int>& devices) : Engine(s, devices, true) {}

private:
    Engine(const ModelSpec& s, const std::vector<int>& devices, bool group) {
        std::vector<int32_t> kind;
        std::vector<double> strike;
        std::vector<uint32_t> mat;
        for (const auto& i : s.instruments) {
            kind.push_back(i.kind == Instrument::Kind::Put ? LTG_PUT : LTG_CALL);
            strike.push_back(i.strike);
            mat.push_back(static_cast<uint32_t>(i.maturity_step));
        }
        ltg_heston_model m{};
        m.mu = s.heston.mu;
        m.s0 = s.heston.s0;
        m.kappa = s.heston.kappa;
        m.theta = s.heston.theta;
        m.xi = s.heston.xi;
        m.rho = s.heston.rho;
        m.v0 = s.heston.v0;
        m.t_nodes = s.grid.t_nodes.data();
        m.n_t_nodes = static_cast<uint32_t>(s.grid.t_nodes.size());
        m.s_nodes = s.grid.s_nodes.data();
        m.n_s_nodes = static_cast<uint32_t>(s.grid.s_nodes.size());
        m.leverage = s.grid.values.data();
        m.inst_kind = kind.data();
        m.inst_strike = strike.data();
        m.inst_maturity_step = mat.data();
        m.n_instruments = static_cast<uint32_t>(kind.size());
        m.steps = static_cast<uint32_t>(s.mc.steps);
        m.dt = s.mc.dt;
        const int rc = group ? ltg_create_heston_devices(&m, devices.data(),
                                                         static_cast<int>(devices.size()), &ctx_)
                             : ltg_create_heston(&m, devices.at(0), &ctx_);
        detail::check(rc, ltg_last_error(nullptr));
    }

public:
    explicit Engine(const ltg_basket_model& m, int device = 0) {
        detail::check(ltg_create_basket(&m, device, &ctx_), ltg_last_error(nullptr));
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { ltg_destroy(ctx_); }

    std::size_t num_params() const { return ltg_num_params(ctx_); }
    std::size_t num_outputs() const { return ltg_num_outputs(ctx_); }
    std::size_t num_randoms() const { return ltg_num_randoms(ctx_); }
    bool rng_exact() const { return ltg_rng_exact(ctx_) != 0; }
    ltg_ctx* handle() const { return ctx_; }

    // expectation.hpp:346-351. Method::tangent replaces pass 2 by pathwise
    // forward tangents (ltg_gradient_of_G_tangent; small-M Heston models).
    enum class Method { adjoint, tangent };
    GradientReport gradient_of_G(std::span<const double> x, std::span<const double> targets,
                                 const MCConfig& cfg, Method method = Method::adjoint) const {
        GradientReport r;
        r.means.resize(num_outputs());
        r.lambda.resize(num_outputs());
        r.grad.resize(num_params());
        ltg_report rep{};
        rep.means = r.means.data();
        rep.lambda = r.lambda.data();
        rep.grad = r.grad.data();
        const ltg_mc_config c = detail::to_c(cfg);
        auto* fn = method == Method::adjoint ? ltg_gradient_of_G : ltg_gradient_of_G_tangent;
        detail::check(fn(ctx_, x.data(), x.size(), targets.data(), targets.size(), &c, &rep),
                      ltg_last_error(ctx_));
        r.G = rep.G;
        r.paths = rep.paths;
        r.seed = rep.seed;
        r.mode = rep.mode == LTG_MODE_STORE ? "store" : "recompute";
        return r;
    }

    // gradient_of_G(kernel, params, targets, src, cfg) with a BufferDrawSource
    // (expectation.hpp:300-344; ltg_gradient_of_G_draws): cfg.seed is echoed,
    // cfg.antithetic unused; fresh_step2_paths reads rows [paths, 2*paths)
    GradientReport gradient_of_G(std::span<const double> x, std::span<const double> targets,
                                 const BufferDraws& src, const MCConfig& cfg) const {
        GradientReport r;
        r.means.resize(num_outputs());
        r.lambda.resize(num_outputs());
        r.grad.resize(num_params());
        ltg_report rep{};
        rep.means = r.means.data();
        rep.lambda = r.lambda.data();
        rep.grad = r.grad.data();
        const ltg_mc_config c = detail::to_c(cfg);
        const ltg_draws d = draws_of(src);
        detail::check(ltg_gradient_of_G_draws(ctx_, x.data(), x.size(), targets.data(),
                                              targets.size(), &d, &c, &rep),
                      ltg_last_error(ctx_));
        r.G = rep.G;
        r.paths = rep.paths;
        r.seed = rep.seed;
        r.mode = rep.mode == LTG_MODE_STORE ? "store" : "recompute";
        return r;
    }

    // the SampleSpace overload (expectation.hpp:354-367)
    GradientReport gradient_of_G(std::span<const double> x, std::span<const double> targets,
                                 const SampleSpace& space) const {
        MCConfig cfg;
        cfg.paths = space.scenarios;
        cfg.seed = 0;
        return gradient_of_G(x, targets, BufferDraws{space.draws, space.num_randoms}, cfg);
    }

    // estimate_means(kernel, params, src, paths) (expectation.hpp:274-279) and
    // the SampleSpace overload (:287-294)
    MeansResult estimate_means(std::span<const double> x, const BufferDraws& src,
                               std::size_t paths) const {
        MeansResult r;
        r.means.resize(num_outputs());
        r.std_errors.resize(num_outputs());
        const ltg_draws d = draws_of(src);
        detail::check(ltg_estimate_means_draws(ctx_, x.data(), x.size(), &d, paths,
                                               r.means.data(), r.std_errors.data()),
                      ltg_last_error(ctx_));
        r.paths = paths;
        return r;
    }
    MeansResult estimate_means(std::span<const double> x, const SampleSpace& space) const {
        return estimate_means(x, BufferDraws{space.draws, space.num_randoms}, space.scenarios);
    }

    // expectation.hpp:281-286
    MeansResult estimate_means(std::span<const double> x, const MCConfig& cfg) const {
        MeansResult r;
        r.means.resize(num_outputs());
        r.std_errors.resize(num_outputs());
        const ltg_mc_config c = detail::to_c(cfg);
        detail::check(ltg_estimate_means(ctx_, x.data(), x.size(), &c, r.means.data(),
                                         r.std_errors.data()),
                      ltg_last_error(ctx_));
        r.paths = cfg.paths;
        return r;
    }

    // expectation.hpp:372-400
    std::vector<double> finite_diff_gradient_of_G(std::span<const double> x,
                                                  std::span<const double> targets,
                                                  const MCConfig& cfg, double h) const {
        std::vector<double> g(num_params());
        const ltg_mc_config c = detail::to_c(cfg);
        detail::check(ltg_finite_diff_gradient_of_G(ctx_, x.data(), x.size(), targets.data(),
                                                    targets.size(), &c, h, g.data()),
                      ltg_last_error(ctx_));
        return g;
    }

    // HBM cap for the checkpoint table + draw store (0: the free memory)
    void set_hbm_budget(std::uint64_t bytes) { detail::check(ltg_set_hbm_budget(ctx_, bytes), ""); }

    // device timing events of the calls (on by default; off for latency-bound loops)
    void set_timing(bool on) { detail::check(ltg_set_timing(ctx_, on ? 1 : 0), ""); }

    // Multi-GPU: rank r of `world` processes (one GPU each) sharing `id`
    // (from nccl_unique_id() on rank 0, broadcast by the caller).
    void attach_nccl(const unsigned char id[128], int rank, int world) {
        detail::check(ltg_attach_nccl(ctx_, id, rank, world), ltg_last_error(ctx_));
    }

private:
    static ltg_draws draws_of(const BufferDraws& src) {
        if (src.dimension == 0 || src.draws.size() % src.dimension != 0)
            throw std::invalid_argument(
                "BufferDrawSource: buffer size not a multiple of dimension");
        return ltg_draws{src.draws.data(), src.draws.size() / src.dimension, src.dimension};
    }

    ltg_ctx* ctx_ = nullptr;
};

inline std::vector<unsigned char> nccl_unique_id() {
    std::vector<unsigned char> id(128);
    detail::check(ltg_nccl_unique_id(id.data()), ltg_last_error(nullptr));
    return id;
}

// The calibrator's plug point (calibrate.hpp:117-120) with common random
// numbers: every evaluation replays cfg.seed. `Report` is the caller's report
// type (lanetape::GradientReport for the reference's gradient_descent).
template <typename Report = GradientReport>
struct ObjectiveT {
    std::function<Report(std::span<const double>)> value_and_grad;
    std::function<double(std::span<const double>)> value;
};

template <typename Report = GradientReport>
ObjectiveT<Report> make_objective(const Engine& e, std::vector<double> targets, MCConfig cfg) {
    ObjectiveT<Report> o;
    o.value_and_grad = [&e, targets, cfg](std::span<const double> x) {
        const GradientReport r = e.gradient_of_G(x, targets, cfg);
        Report out;
        out.G = r.G;
        out.means = r.means;
        out.lambda = r.lambda;
        out.grad = r.grad;
        out.paths = r.paths;
        out.mode = r.mode;
        out.seed = r.seed;
        return out;
    };
    o.value = [&e, targets, cfg](std::span<const double> x) {
        const MeansResult m = e.estimate_means(x, cfg);
        double G = 0.0;
        for (std::size_t i = 0; i < targets.size(); ++i) {
            const double l = m.means[i] - targets[i];
            G += 0.5 * l * l;
        }
        return G;
    };
    return o;
}

}  // namespace lanetape_b200
