// oracle/ref_driver.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A C-ABI shim over the UNMODIFIED reference library (`lanetape`, header-only
// C++20 under /root/reference/proj/include). It is compiled from those
// headers in place by oracle/Makefile into oracle/_ref/libltref.so (git-
// ignored, shipped to the GPU box with the snapshot). Only tests/, the
// smoke() check and bench.py's CPU-baseline / reference arm may load it.
//
// Every function forwards to the reference's own code path:
//   ltref_philox_block        Philox4x32::block              rng.hpp:19-31
//   ltref_uniform             uniform_from_bits              rng.hpp:38-40
//   ltref_inverse_normal_cdf  inverse_normal_cdf             rng.hpp:45-85
//   ltref_fill_normals        PhiloxNormalSource::fill       rng.hpp:113-127
//   ltref_record_heston       record_heston_program          heston.hpp:245-325
//   ltref_record_basket       a program recorded with the public Tape API
//                             (config 4 has no model in the reference layer)
//   ltref_gradient_of_G       gradient_of_G(Kernel, ...)     expectation.hpp:300-344
//   ltref_estimate_means      estimate_means                 expectation.hpp:274-286
//   ltref_forward_sums        detail::forward_pass           expectation.hpp:152-198
//   ltref_reverse_sums        detail::reverse_pass           expectation.hpp:204-249
//   ltref_path_adjoint        forward_eval + reverse_seeded  tape.hpp:276-413
//   ltref_simulate_path       HestonSimulator::simulate_path heston.hpp:385-424
//   ltref_finite_diff_gradient_of_G                           expectation.hpp:372-400
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.h"

using namespace lanetape;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const EvalError& e) {
        return fail(e, 2);
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 4);
    }
}

struct Program {
    Tape tape;
    std::vector<double> initial;
    // scalar simulator for Heston programs (cost(F) / parity of the tape)
    std::unique_ptr<HestonSimulator> sim;
};

ModelSpec heston_spec(const ltg_heston_model& m) {
    ModelSpec s;
    s.heston.mu = m.mu;
    s.heston.s0 = m.s0;
    s.heston.kappa = m.kappa;
    s.heston.theta = m.theta;
    s.heston.xi = m.xi;
    s.heston.rho = m.rho;
    s.heston.v0 = m.v0;
    s.grid.t_nodes.assign(m.t_nodes, m.t_nodes + m.n_t_nodes);
    s.grid.s_nodes.assign(m.s_nodes, m.s_nodes + m.n_s_nodes);
    s.grid.values.assign(m.leverage, m.leverage + std::size_t(m.n_t_nodes) * m.n_s_nodes);
    for (uint32_t i = 0; i < m.n_instruments; ++i) {
        Instrument ins;
        ins.kind = m.inst_kind[i] == LTG_PUT ? Instrument::Kind::Put : Instrument::Kind::Call;
        ins.strike = m.inst_strike[i];
        ins.maturity_step = m.inst_maturity_step[i];
        s.instruments.push_back(ins);
    }
    s.mc.paths = 1;
    s.mc.steps = m.steps;
    s.mc.dt = m.dt;
    s.mc.seed = 0;
    return s;
}

// Config-4 program: n correlated log-Euler GBMs. The recording order below IS
// the definition of the model's arithmetic; the GPU kernel restates it
// (paper_1901_04200_b200/csrc/basket.cu). Per asset a, hoisted:
//   drift_a = (r - 0.5*(sigma_a*sigma_a)) * dt,  vol_a = sigma_a * sqrt(dt)
// per step k:  w_a = ((L[a][0]*z0 + L[a][1]*z1) + ...) + L[a][a]*z_a
//              S_a = S_a * exp(drift_a + vol_a * w_a)
// payoff of instrument i on asset a at maturity_step: max(+-(S_a - K), 0).
void record_basket(const ltg_basket_model& m, Program& p) {
    if (m.n_assets == 0 || m.steps == 0 || !(m.dt > 0.0) || m.n_instruments == 0)
        throw std::invalid_argument("basket: empty model");
    Tape& T = p.tape;
    const uint32_t n = m.n_assets;
    std::vector<VarId> sigma(n);
    for (uint32_t a = 0; a < n; ++a) {
        sigma[a] = T.new_input(InputKind::Parameter, m.sigma[a]);
        p.initial.push_back(m.sigma[a]);
    }
    std::vector<VarId> z;
    for (uint32_t k = 0; k < m.steps * n; ++k) z.push_back(T.new_input(InputKind::Random, 0.0));
    const VarId c_r = T.constant(m.r);
    const VarId c_half = T.constant(0.5);
    const VarId c_dt = T.constant(m.dt);
    const VarId c_sqdt = T.constant(std::sqrt(m.dt));
    std::vector<VarId> drift(n), vol(n), S(n);
    for (uint32_t a = 0; a < n; ++a) {
        drift[a] = T.mul(T.sub(c_r, T.mul(c_half, T.mul(sigma[a], sigma[a]))), c_dt);
        vol[a] = T.mul(sigma[a], c_sqdt);
        S[a] = T.constant(m.s0[a]);
    }
    std::vector<std::vector<VarId>> s_at(m.steps + 1, std::vector<VarId>(n));
    s_at[0] = S;
    for (uint32_t k = 0; k < m.steps; ++k) {
        for (uint32_t a = 0; a < n; ++a) {
            VarId w = T.mul(T.constant(m.chol[a * n + 0]), z[k * n + 0]);
            for (uint32_t b = 1; b <= a; ++b)
                w = T.add(w, T.mul(T.constant(m.chol[a * n + b]), z[k * n + b]));
            S[a] = T.mul(S[a], T.exp(T.add(drift[a], T.mul(vol[a], w))));
        }
        s_at[k + 1] = S;
    }
    for (uint32_t i = 0; i < m.n_instruments; ++i) {
        if (m.inst_asset[i] >= n || m.inst_maturity_step[i] == 0 ||
            m.inst_maturity_step[i] > m.steps)
            throw std::invalid_argument("basket: bad instrument");
        const VarId s_mat = s_at[m.inst_maturity_step[i]][m.inst_asset[i]];
        const VarId K = T.constant(m.inst_strike[i]);
        const VarId pay = m.inst_kind[i] == LTG_PUT ? T.max_zero(T.sub(K, s_mat))
                                                     : T.max_zero(T.sub(s_mat, K));
        T.mark_output(pay);
    }
}

}  // namespace

extern "C" {

const char* ltref_last_error(void) { return g_err.c_str(); }

void ltref_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const auto r = Philox4x32::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

double ltref_uniform(uint32_t w0, uint32_t w1) { return uniform_from_bits(w0, w1); }

int ltref_inverse_normal_cdf(double p, double* out) {
    return guarded([&] {
        try {
            *out = inverse_normal_cdf(p);
        } catch (const std::domain_error& e) {
            throw std::invalid_argument(e.what());
        }
    });
}

int ltref_fill_normals(uint64_t seed, size_t dim, int antithetic, uint64_t path0, uint64_t npaths,
                       double* out) {
    return guarded([&] {
        PhiloxNormalSource src(seed, dim, antithetic != 0);
        for (uint64_t p = 0; p < npaths; ++p)
            src.fill(path0 + p, std::span<double>(out + p * dim, dim));
    });
}

void* ltref_record_heston(const ltg_heston_model* m) {
    try {
        auto p = std::make_unique<Program>();
        ModelSpec s = heston_spec(*m);
        HestonProgram hp = record_heston_program(s.heston, s.grid, s.instruments, s.mc.steps, s.mc.dt);
        p->tape = std::move(hp.tape);
        p->initial = hp.initial_params;
        p->sim = std::make_unique<HestonSimulator>(s.heston, s.grid, s.instruments, s.mc.steps,
                                                   s.mc.dt);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ltref_record_basket(const ltg_basket_model* m) {
    try {
        auto p = std::make_unique<Program>();
        record_basket(*m, *p);
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// y = x * w, the hand-checked linear case of test_expectation.cpp:113-134
void* ltref_record_linear(void) {
    auto p = std::make_unique<Program>();
    const VarId x = p->tape.new_input(InputKind::Parameter, 1.0);
    const VarId w = p->tape.new_input(InputKind::Random, 0.0);
    p->tape.mark_output(p->tape.mul(x, w));
    p->initial = {1.0};
    return p.release();
}

void ltref_free(void* prog) { delete static_cast<Program*>(prog); }

size_t ltref_num_params(void* prog) { return static_cast<Program*>(prog)->tape.num_params(); }
size_t ltref_num_randoms(void* prog) { return static_cast<Program*>(prog)->tape.num_randoms(); }
size_t ltref_num_outputs(void* prog) { return static_cast<Program*>(prog)->tape.num_outputs(); }
size_t ltref_num_nodes(void* prog) { return static_cast<Program*>(prog)->tape.size(); }
void ltref_initial_params(void* prog, double* x) {
    auto* p = static_cast<Program*>(prog);
    std::copy(p->initial.begin(), p->initial.end(), x);
}

static MCConfig make_cfg(uint64_t paths, uint64_t seed, int antithetic, int lane_width, int workers,
                         int memory_mode, int fresh) {
    MCConfig cfg;
    cfg.paths = paths;
    cfg.seed = seed;
    cfg.antithetic = antithetic != 0;
    cfg.lane_width = lane_width;
    cfg.worker_threads = workers;
    cfg.memory_mode = memory_mode == LTG_MODE_STORE ? MemoryMode::Store : MemoryMode::Recompute;
    cfg.fresh_step2_paths = fresh != 0;
    return cfg;
}

int ltref_gradient_of_G(void* prog, const double* x, size_t M, const double* C, size_t m,
                        uint64_t paths, uint64_t seed, int antithetic, int lane_width, int workers,
                        int memory_mode, int fresh, double* G, double* means, double* lambda,
                        double* grad) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        MCConfig cfg = make_cfg(paths, seed, antithetic, lane_width, workers, memory_mode, fresh);
        auto rep = gradient_of_G(p->tape, std::span<const double>(x, M),
                                 std::span<const double>(C, m), cfg);
        *G = rep.G;
        std::copy(rep.means.begin(), rep.means.end(), means);
        std::copy(rep.lambda.begin(), rep.lambda.end(), lambda);
        std::copy(rep.grad.begin(), rep.grad.end(), grad);
    });
}

// gradient_of_G over an explicit scenario set (expectation.hpp:354-367)
int ltref_gradient_of_G_space(void* prog, const double* x, size_t M, const double* C, size_t m,
                              const double* draws, size_t scenarios, int lane_width, double* G,
                              double* means, double* lambda, double* grad) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        SampleSpace space;
        space.scenarios = scenarios;
        space.num_randoms = p->tape.num_randoms();
        space.draws.assign(draws, draws + scenarios * space.num_randoms);
        auto rep = gradient_of_G(p->tape, std::span<const double>(x, M),
                                 std::span<const double>(C, m), space, lane_width);
        *G = rep.G;
        std::copy(rep.means.begin(), rep.means.end(), means);
        std::copy(rep.lambda.begin(), rep.lambda.end(), lambda);
        std::copy(rep.grad.begin(), rep.grad.end(), grad);
    });
}

// gradient_of_G(Kernel, params, targets, PathDrawSource, cfg) with a
// BufferDrawSource over the caller's path-major rows (expectation.hpp:300-344,
// rng.hpp:140-167): the reference side of ltg_gradient_of_G_draws
int ltref_gradient_of_G_buffer(void* prog, const double* x, size_t M, const double* C, size_t m,
                               const double* draws, size_t rows, uint64_t paths, int fresh,
                               int memory_mode, int lane_width, int workers, double* G,
                               double* means, double* lambda, double* grad) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        const size_t dim = p->tape.num_randoms();
        BufferDrawSource src(std::vector<double>(draws, draws + rows * dim), dim);
        MCConfig cfg = make_cfg(paths, 0, 0, lane_width, workers, memory_mode, fresh);
        Kernel k = Kernel::freeze(p->tape, lane_width);
        auto rep = gradient_of_G(k, std::span<const double>(x, M), std::span<const double>(C, m),
                                 src, cfg);
        *G = rep.G;
        std::copy(rep.means.begin(), rep.means.end(), means);
        std::copy(rep.lambda.begin(), rep.lambda.end(), lambda);
        std::copy(rep.grad.begin(), rep.grad.end(), grad);
    });
}

// estimate_means(Kernel, params, PathDrawSource, paths, workers) over a
// BufferDrawSource (expectation.hpp:274-279)
int ltref_estimate_means_buffer(void* prog, const double* x, size_t M, const double* draws,
                                size_t rows, uint64_t paths, int lane_width, int workers,
                                double* means, double* se) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        const size_t dim = p->tape.num_randoms();
        BufferDrawSource src(std::vector<double>(draws, draws + rows * dim), dim);
        Kernel k = Kernel::freeze(p->tape, lane_width);
        auto r = estimate_means(k, std::span<const double>(x, M), src, paths, workers);
        std::copy(r.means.begin(), r.means.end(), means);
        if (se) std::copy(r.std_errors.begin(), r.std_errors.end(), se);
    });
}

int ltref_estimate_means(void* prog, const double* x, size_t M, uint64_t paths, uint64_t seed,
                         int antithetic, int lane_width, int workers, double* means, double* se) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        MCConfig cfg = make_cfg(paths, seed, antithetic, lane_width, workers, 0, 0);
        auto r = estimate_means(p->tape, std::span<const double>(x, M), cfg);
        std::copy(r.means.begin(), r.means.end(), means);
        if (se) std::copy(r.std_errors.begin(), r.std_errors.end(), se);
    });
}

int ltref_forward_sums(void* prog, const double* x, size_t M, uint64_t seed, int antithetic,
                       int lane_width, int workers, uint64_t path_offset, uint64_t paths,
                       double* sum, double* sumsq) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        Kernel k = Kernel::freeze(p->tape, lane_width);
        PhiloxNormalSource src(seed, p->tape.num_randoms(), antithetic != 0);
        auto r = detail::forward_pass(k, std::span<const double>(x, M), src, path_offset, paths,
                                      workers, false);
        std::copy(r.sum.begin(), r.sum.end(), sum);
        std::copy(r.sumsq.begin(), r.sumsq.end(), sumsq);
    });
}

int ltref_reverse_sums(void* prog, const double* x, size_t M, uint64_t seed, int antithetic,
                       int lane_width, int workers, uint64_t path_offset, uint64_t paths,
                       const double* lambda, size_t m, double* total) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        Kernel k = Kernel::freeze(p->tape, lane_width);
        PhiloxNormalSource src(seed, p->tape.num_randoms(), antithetic != 0);
        auto t = detail::reverse_pass(k, std::span<const double>(x, M), src, path_offset, paths,
                                      workers, std::span<const double>(lambda, m), nullptr);
        std::copy(t.begin(), t.end(), total);
    });
}

// One path: outputs y (m) and the parameter adjoints of lambda.y (M).
int ltref_path_adjoint(void* prog, const double* x, size_t M, const double* draws, size_t N,
                       const double* lambda, size_t m, double* y, double* adj) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        EvalState st;
        auto out = forward_eval(p->tape, std::span<const double>(x, M),
                                std::span<const double>(draws, N), st);
        std::copy(out.begin(), out.end(), y);
        if (adj) {
            auto a = reverse_seeded(p->tape, st, std::span<const double>(lambda, m));
            std::copy(a.begin(), a.begin() + M, adj);
        }
    });
}

int ltref_simulate_path(void* prog, const double* x, size_t M, const double* draws, size_t N,
                        double* payoffs) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        if (!p->sim) throw std::invalid_argument("simulate_path: not a Heston program");
        p->sim->set_params(std::span<const double>(x, M));
        p->sim->simulate_path(std::span<const double>(draws, N),
                              std::span<double>(payoffs, p->tape.num_outputs()));
    });
}

int ltref_finite_diff_gradient_of_G(void* prog, const double* x, size_t M, const double* C,
                                    size_t m, uint64_t paths, uint64_t seed, int lane_width,
                                    int workers, double h, double* grad) {
    return guarded([&] {
        auto* p = static_cast<Program*>(prog);
        MCConfig cfg = make_cfg(paths, seed, 0, lane_width, workers, 0, 0);
        auto g = finite_diff_gradient_of_G(p->tape, std::span<const double>(x, M),
                                           std::span<const double>(C, m), cfg, h);
        std::copy(g.begin(), g.end(), grad);
    });
}

}  // extern "C"
