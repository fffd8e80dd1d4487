// examples/lanetape_gpu.cpp — the reference CLI's `price`, `gradcheck` and
// `calibrate` commands (P/tools/main.cpp:134-382) with the Monte Carlo on the
// B200 engine (the calibrator and the artifacts with the
// echoed config). `bench` (the CPU cost-coefficient benchmark) is out of scope.
//
// Same flags, same artifact files and key order (price.json, gradcheck.json:
// {"config": {"command", "model", "run"}, <report fields>}), same exit codes
// (0 ok, 1 validation/usage, 2 numerical). The model JSON is read and echoed
// by the reference's own lanetape::load_model_spec / to_json (compiled in
// place); estimate_means, gradient_of_G and finite_diff_gradient_of_G run on
// the GPU through lanetape_b200.hpp. lane_width / threads / memory_mode are
// the reference's CPU knobs: accepted, echoed, and without effect on the GPU.
//
// Usage: lanetape_gpu price|gradcheck|calibrate --config model.json [--out-dir D]
//        [--seed S] [--paths P] [--lane-width W] [--threads T]
//        [--memory-mode recompute|store]
//        gradcheck: [--fd-h H] [--tolerance TOL]
//        calibrate: [--free kappa,theta,...|leverage] [--init name=value]...
//                   [--init-factor F] [--max-iters N] [--g-rel-tol T] [--initial-step S]
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.hpp"
#include "lanetape_b200_ref.hpp"

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
    // calibrate (main.cpp:236-245)
    std::string free_params = "kappa,theta";
    std::vector<std::string> init;
    double init_factor = 1.5;
    std::size_t max_iters = 500;
    double g_rel_tol = 1e-10;
    double initial_step = 1.0;
};

Opts parse(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: lanetape_gpu price|gradcheck --config F");
    Opts o;
    o.command = argv[1];
    if (o.command != "price" && o.command != "gradcheck" && o.command != "calibrate")
        throw std::invalid_argument("unknown command '" + o.command +
                                    "' (price, gradcheck, calibrate)");
    const bool cal = o.command == "calibrate";
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
        else if (flag == "--free" && cal) o.free_params = v;
        else if (flag == "--init" && cal) o.init.push_back(v);
        else if (flag == "--init-factor" && cal) o.init_factor = std::stod(v);
        else if (flag == "--max-iters" && cal) o.max_iters = std::stoull(v);
        else if (flag == "--g-rel-tol" && cal) o.g_rel_tol = std::stod(v);
        else if (flag == "--initial-step" && cal) o.initial_step = std::stod(v);
        else throw std::invalid_argument("unknown option " + flag);
    }
    if (o.config_path.empty()) throw std::invalid_argument("--config is required");
    if (o.memory_mode != "recompute" && o.memory_mode != "store")
        throw std::invalid_argument("--memory-mode: recompute or store");
    return o;
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
    gpu::Engine engine(gpu::to_gpu(spec));
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
    gpu::Engine engine(gpu::to_gpu(spec));
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

const std::array<std::string, lt::heston_free_params> scalar_names{"kappa", "theta", "xi", "rho",
                                                                   "v0"};

std::vector<std::string> param_names(const lt::LeverageGrid& g) {
    std::vector<std::string> names(scalar_names.begin(), scalar_names.end());
    for (std::size_t r = 0; r < g.rows(); ++r)
        for (std::size_t c = 0; c < g.cols(); ++c)
            names.push_back("L_" + std::to_string(r) + "_" + std::to_string(c));
    return names;
}

std::vector<std::string> split_csv(const std::string& s) {
    std::vector<std::string> out;
    std::istringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ','))
        if (!tok.empty()) out.push_back(tok);
    return out;
}

// main.cpp:256-382: gradient_descent (unchanged, the reference's) on synthetic
// targets at the truth, descending in truth-scaled coordinates
int run_calibrate(const Opts& o, const lt::ModelSpec& spec) {
    gpu::Engine engine(gpu::to_gpu(spec));
    const gpu::MCConfig cfg = mc_config(spec, o);
    const std::vector<double> truth = lt::pack_params(spec.heston, spec.grid);
    const std::size_t M = truth.size();
    const auto names = param_names(spec.grid);

    lt::Bounds bounds{truth, truth};  // frozen at the truth unless named in --free
    const std::array<std::pair<double, double>, lt::heston_free_params> scalar_box{
        {{1e-3, 25.0}, {1e-5, 4.0}, {0.0, 5.0}, {-0.995, 0.995}, {1e-5, 4.0}}};
    std::vector<bool> is_free(M, false);
    for (const auto& tok : split_csv(o.free_params)) {
        bool matched = false;
        for (std::size_t j = 0; j < lt::heston_free_params; ++j)
            if (tok == scalar_names[j]) {
                bounds.lo[j] = scalar_box[j].first;
                bounds.hi[j] = scalar_box[j].second;
                is_free[j] = true;
                matched = true;
            }
        if (tok == "leverage") {
            for (std::size_t j = lt::heston_free_params; j < M; ++j) {
                bounds.lo[j] = 1e-3;
                bounds.hi[j] = 10.0;
                is_free[j] = true;
            }
            matched = true;
        }
        if (!matched)
            throw std::invalid_argument("calibrate: unknown --free token '" + tok +
                                        "' (expected kappa, theta, xi, rho, v0 or leverage)");
    }
    if (std::none_of(is_free.begin(), is_free.end(), [](bool b) { return b; }))
        throw std::invalid_argument("calibrate: --free selected no parameters");

    std::vector<double> x0(truth);
    for (std::size_t j = 0; j < M; ++j)
        if (is_free[j]) x0[j] = truth[j] * o.init_factor;
    for (const auto& kv : o.init) {
        const auto eq = kv.find('=');
        if (eq == std::string::npos)
            throw std::invalid_argument("calibrate: --init expects name=value, got '" + kv + "'");
        const std::string name = kv.substr(0, eq);
        const auto it = std::find(names.begin(), names.end(), name);
        if (it == names.end())
            throw std::invalid_argument("calibrate: unknown parameter '" + name + "'");
        x0[static_cast<std::size_t>(it - names.begin())] = std::stod(kv.substr(eq + 1));
    }
    bounds.project(x0);

    // synthetic_targets (calibrate.hpp:224-227) on the GPU
    const std::vector<double> targets = engine.estimate_means(truth, cfg).means;
    require_finite(targets, "calibrate targets");
    const auto g = gpu::make_objective<lt::GradientReport>(engine, targets, cfg);
    lt::Objective objective{g.value_and_grad, g.value};

    lt::OptimizerConfig opt;
    opt.max_iters = o.max_iters;
    opt.g_rel_tol = o.g_rel_tol;
    opt.initial_step = o.initial_step;
    opt.scales.resize(M);
    for (std::size_t j = 0; j < M; ++j) opt.scales[j] = std::max(std::abs(truth[j]), 1e-2);
    const lt::CalibrationResult res = lt::gradient_descent(objective, x0, bounds, opt);
    require_finite(res.params, "calibrate parameters");

    const auto config = effective_config(o, spec);
    nlohmann::ordered_json body;
    body["converged"] = res.converged;
    body["stop_reason"] = res.stop_reason;
    body["iters"] = res.iters;
    body["G"] = res.G;
    body["targets"] = targets;
    nlohmann::ordered_json fitted, truth_j, start_j;
    for (std::size_t j = 0; j < M; ++j) {
        if (!is_free[j]) continue;
        fitted[names[j]] = res.params[j];
        truth_j[names[j]] = truth[j];
        start_j[names[j]] = x0[j];
    }
    body["fitted"] = fitted;
    body["truth"] = truth_j;
    body["start"] = start_j;
    write_artifact(o, "calibrate.json", config, body);
    std::ostringstream csv;
    csv << "# config: " << config.dump() << "\n";
    res.trajectory.write_csv(csv, names);
    {
        const auto path = std::filesystem::path(o.out_dir) / "trajectory.csv";
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::invalid_argument("cannot write " + path.string());
        out << csv.str();
        std::cout << "wrote " << path.string() << "\n";
    }
    std::cout << "calibrate: " << res.stop_reason << " after " << res.iters << " iterations, G "
              << res.G << "\n";
    for (std::size_t j = 0; j < M; ++j)
        if (is_free[j])
            std::cout << "  " << names[j] << ": " << res.params[j] << " (truth " << truth[j]
                      << ")\n";
    return exit_ok;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Opts o = parse(argc, argv);
        lt::ModelSpec spec = lt::load_model_spec(o.config_path);
        if (o.seed) spec.mc.seed = *o.seed;
        if (o.paths) spec.mc.paths = *o.paths;
        lt::validate(spec);
        if (o.command == "price") return run_price(o, spec);
        if (o.command == "gradcheck") return run_gradcheck(o, spec);
        return run_calibrate(o, spec);
    } catch (const gpu::EvalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return exit_numerical;
    } catch (const lt::EvalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return exit_numerical;
    } catch (const nlohmann::json::exception& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return exit_validation;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return exit_validation;
    }
}
