// lanetape_b200_ref.hpp — the glue a reference user adds: the reference's own
// model types (lanetape/heston.hpp, compiled in place) converted to the
// engine's mirror types (lanetape_b200.hpp). Include after the reference
// headers; header-only.
//
//   lanetape::ModelSpec spec = lanetape::load_model_spec("model.json");
//   auto engine = lanetape_b200::make_engine(spec);        // ~ record_heston_program
//   auto report = engine.gradient_of_G(x, targets, lanetape_b200::mc_config(spec));
#pragma once

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.hpp"

namespace lanetape_b200 {

// field-by-field copy of ModelSpec (L/heston.hpp:20-114)
inline ModelSpec to_gpu(const lanetape::ModelSpec& s) {
    ModelSpec g;
    g.heston = {s.heston.mu, s.heston.kappa, s.heston.theta, s.heston.xi,
                s.heston.rho, s.heston.v0,   s.heston.s0};
    g.grid = {s.grid.t_nodes, s.grid.s_nodes, s.grid.values};
    for (const auto& i : s.instruments)
        g.instruments.push_back({i.kind == lanetape::Instrument::Kind::Put ? Instrument::Kind::Put
                                                                         : Instrument::Kind::Call,
                                 i.strike, i.maturity_step});
    g.mc = {s.mc.paths, s.mc.steps, s.mc.dt, s.mc.seed};
    return g;
}

// MCConfig (L/expectation.hpp:25-39) with the spec's paths and seed
inline MCConfig mc_config(const lanetape::ModelSpec& s) {
    MCConfig c;
    c.paths = s.mc.paths;
    c.seed = s.mc.seed;
    return c;
}

inline MCConfig to_gpu(const lanetape::MCConfig& r) {
    MCConfig c;
    c.paths = r.paths;
    c.seed = r.seed;
    c.antithetic = r.antithetic;
    c.lane_width = static_cast<int>(r.lane_width);
    c.worker_threads = static_cast<int>(r.worker_threads);
    c.memory_mode = r.memory_mode == lanetape::MemoryMode::Store ? MemoryMode::Store
                                                                  : MemoryMode::Recompute;
    c.fresh_step2_paths = r.fresh_step2_paths;
    c.store_limit_bytes = r.store_limit_bytes;
    return c;
}

inline Engine make_engine(const lanetape::ModelSpec& s, int device = 0) {
    return Engine(to_gpu(s), device);
}

}  // namespace lanetape_b200
