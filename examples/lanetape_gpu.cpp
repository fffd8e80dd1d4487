// examples/lanetape_gpu.cpp — the reference CLI's `price` and `gradcheck`
// commands (P/tools/main.cpp:134-205) with the Monte Carlo on the B200
// engine (the artifacts with the echoed config).
//
// Same flags, same artifact files and key order (price.json, gradcheck.json:
// {"config": {"command", "model", "run"}, <report fields>}), same exit codes
// (0 ok, 1 validation/usage, 2 numerical). The model JSON is read and echoed
// by the reference's own lanetape::load_model_spec / to_json (compiled in
// place); estimate_means, gradient_of_G and finite_diff_gradient_of_G run on
// the GPU through lanetape_b200.hpp. lane_width / threads / memory_mode are
// the reference's CPU knobs: accepted, echoed, and without effect on the GPU.
//
// Usage: lanetape_gpu price|gradcheck --config model.json [--out-dir D]
//        [--seed S] [--paths P] [--lane-width W] [--threads T]
//        [--memory-mode recompute|store] [--fd-h H] [--tolerance TOL]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.hpp"

namespace lt = lanetape;
namespace gpu = lanetape_b200;

namespace {

constexpr int exit_ok = 0;
constexpr int exit_validation = 1;
constexpr int exit_numerical = 2;

struct Opts {
    std::string command;
    std::string config_path;
    std::string out_dir = ".";
    std::optional<std::uint64_t> seed;
    std::optional<std::size_t> paths;
    int lane_width = 4;
    int threads = 1;
    std::string memory_mode = "recompute";
    double fd_h = 3e-7;  // the reference's gradcheck defaults (main.cpp:126-132)
    double tolerance = 1e-6;
};

Opts parse(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: lanetape_gpu price|gradcheck --config F");
    Opts o;
    o.command = argv[1];
    if (o.command != "price" && o.command != "gradcheck")
        throw std::invalid_argument("unknown command '" + o.command + "' (price, gradcheck)");
    for (int i = 2; i < argc; ++i) {
        const std::string flag = argv[i];
        if (i + 1 >= argc) throw std::invalid_argument(flag + " needs a value");
        const std::string v = argv[++i];
        if (flag == "--config") o.config_path = v;
        else if (flag == "--out-dir") o.out_dir = v;
        else if (flag == "--seed") o.seed = std::stoull(v);
        else if (flag == "--paths") o.paths = std::stoull(v);
        else if (flag == "--lane-width") o.lane_width = std::stoi(v);
        else if (flag == "--threads") o.threads = std::stoi(v);
        else if (flag == "--memory-mode") o.memory_mode = v;
        else if (flag == "--fd-h" && o.command == "gradcheck") o.fd_h = std::stod(v);
        else if (flag == "--tolerance" && o.command == "gradcheck") o.tolerance = std::stod(v);
        else throw std::invalid_argument("unknown option " + flag);
    }
    if (o.config_path.empty()) throw std::invalid_argument("--config is required");
    if (o.memory_mode != "recompute" && o.memory_mode != "store")
        throw std::invalid_argument("--memory-mode: recompute or store");
    return o;
}

gpu::ModelSpec to_gpu(const lt::ModelSpec& s) {
    gpu::ModelSpec g;
    g.heston = {s.heston.mu, s.heston.kappa, s.heston.theta, s.heston.xi,
                s.heston.rho, s.heston.v0,   s.heston.s0};
    g.grid = {s.grid.t_nodes, s.grid.s_nodes, s.grid.values};
    for (const auto& i : s.instruments)
        g.instruments.push_back({i.kind == lt::Instrument::Kind::Put ? gpu::Instrument::Kind::Put
                                                                     : gpu::Instrument::Kind::Call,
                                 i.strike, i.maturity_step});
    g.mc = {s.mc.paths, s.mc.steps, s.mc.dt, s.mc.seed};
    return g;
}

// main.cpp:72-81
nlohmann::ordered_json effective_config(const Opts& o, const lt::ModelSpec& spec) {
    nlohmann::ordered_json j;
    j["command"] = o.command;
    j["model"] = lt::to_json(spec);
    j["run"] = {{"lane_width", o.lane_width},
                {"worker_threads", o.threads},
                {"memory_mode", o.memory_mode}};
    return j;
}

// main.cpp:97-103: the echoed config first, then the report fields
void write_artifact(const Opts& o, const char* name, const nlohmann::ordered_json& config,
                    const nlohmann::ordered_json& body) {
    std::filesystem::path dir(o.out_dir);
    std::filesystem::create_directories(dir);
    nlohmann::ordered_json j;
    j["config"] = config;
    for (const auto& [key, value] : body.items()) j[key] = value;
    const auto path = dir / name;
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::invalid_argument("cannot write " + path.string());
    out << j.dump(2) << "\n";
    std::cout << "wrote " << path.string() << "\n";
}

void require_finite(const std::vector<double>& xs, const char* what) {
    for (double x : xs)
        if (!std::isfinite(x)) throw gpu::EvalError(std::string(what) + ": non-finite result");
}

gpu::MCConfig mc_config(const lt::ModelSpec& spec, const Opts& o) {
    gpu::MCConfig cfg;
    cfg.paths = spec.mc.paths;
    cfg.seed = spec.mc.seed;
    cfg.lane_width = o.lane_width;
    cfg.worker_threads = o.threads;
    cfg.memory_mode = o.memory_mode == "store" ? gpu::MemoryMode::Store : gpu::MemoryMode::Recompute;
    return cfg;
}

int run_price(const Opts& o, const lt::ModelSpec& spec) {
    gpu::Engine engine(to_gpu(spec));
    const std::vector<double> x = lt::pack_params(spec.heston, spec.grid);
    const auto means = engine.estimate_means(x, mc_config(spec, o));
    require_finite(means.means, "price means");
    nlohmann::ordered_json body;
    body["means"] = means.means;
    body["std_errors"] = means.std_errors;
    body["paths"] = means.paths;
    body["seed"] = spec.mc.seed;
    write_artifact(o, "price.json", effective_config(o, spec), body);
    for (std::size_t i = 0; i < means.means.size(); ++i)
        std::cout << "instrument " << i << ": mean " << means.means[i] << " (se "
                  << means.std_errors[i] << ")\n";
    return exit_ok;
}

// main.cpp:134-182: targets are 90% of the means at the config parameters
int run_gradcheck(const Opts& o, const lt::ModelSpec& spec) {
    gpu::Engine engine(to_gpu(spec));
    const gpu::MCConfig cfg = mc_config(spec, o);
    const std::vector<double> x = lt::pack_params(spec.heston, spec.grid);
    const auto means = engine.estimate_means(x, cfg);
    require_finite(means.means, "gradcheck means");
    std::vector<double> targets(means.means.size());
    for (std::size_t i = 0; i < targets.size(); ++i) targets[i] = 0.9 * means.means[i];

    const auto report = engine.gradient_of_G(x, targets, cfg);
    require_finite(report.grad, "gradcheck gradient");
    const auto fd = engine.finite_diff_gradient_of_G(x, targets, cfg, o.fd_h);
    require_finite(fd, "gradcheck finite differences");

    double max_rel = 0.0;
    std::vector<double> rel(report.grad.size());
    for (std::size_t j = 0; j < report.grad.size(); ++j) {
        const double denom = std::max(std::fabs(report.grad[j]), 1e-8);
        rel[j] = std::fabs(report.grad[j] - fd[j]) / denom;
        max_rel = std::max(max_rel, rel[j]);
    }
    const bool pass = max_rel <= o.tolerance;
    nlohmann::ordered_json body;
    body["h"] = o.fd_h;
    body["tolerance"] = o.tolerance;
    body["max_rel_err"] = max_rel;
    body["pass"] = pass;
    body["G"] = report.G;
    body["grad"] = report.grad;
    body["fd_grad"] = fd;
    body["rel_err"] = rel;
    write_artifact(o, "gradcheck.json", effective_config(o, spec), body);
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.3e", max_rel);
    std::cout << "gradcheck: max rel err " << buf << " over " << report.grad.size()
              << " parameters, tolerance " << o.tolerance << " -> " << (pass ? "PASS" : "FAIL")
              << "\n";
    return pass ? exit_ok : exit_validation;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Opts o = parse(argc, argv);
        lt::ModelSpec spec = lt::load_model_spec(o.config_path);
        if (o.seed) spec.mc.seed = *o.seed;
        if (o.paths) spec.mc.paths = *o.paths;
        lt::validate(spec);
        return o.command == "price" ? run_price(o, spec) : run_gradcheck(o, spec);
    } catch (const gpu::EvalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return exit_numerical;
    } catch (const lt::EvalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return exit_numerical;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    }
}
