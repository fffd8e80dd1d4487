// examples/lanetape_gpu.cpp — `price` and `gradcheck` runs of a ModelSpec file
// with the Monte Carlo on the B200 engine, writing the JSON artifacts a
// reference user's tooling reads.
//
// Artifact schema (pinned by tests/test_cli_gpu.py): one object per run,
//   {"config": {"command", "model", "run"}, <results>}
// where "model" is the ModelSpec as the reference serialises it
// (lanetape::to_json, heston.hpp) with --paths / --seed applied, and "run" the
// reference's CPU knobs {"lane_width", "worker_threads", "memory_mode"}
// (accepted and echoed; they do not change the GPU computation).
//   price.json      results: means, std_errors, paths, seed
//   gradcheck.json  results: h, tolerance, max_rel_err, pass, G, grad, fd_grad, rel_err
//                   (targets = 0.9 * means; adjoint vs central differences under
//                   common random numbers, rel err with a 1e-8 denominator floor)
// Exit status: 0 ok, 1 bad usage / invalid input / gradcheck above tolerance,
// 2 non-finite result (the reference's EvalError class of failure).
//
// usage: lanetape_gpu price|gradcheck --config model.json [--out-dir D] [--seed S]
//        [--paths P] [--lane-width W] [--threads T] [--memory-mode recompute|store]
//        [--fd-h H] [--tolerance TOL]          (the last two: gradcheck only)
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "lanetape/lanetape.hpp"
#include "lanetape_b200.hpp"
#include "lanetape_b200_ref.hpp"

namespace gpu = lanetape_b200;
using Json = nlohmann::ordered_json;

namespace {

struct Usage : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct Run {
    std::string command, config, out_dir = ".", memory_mode = "recompute";
    long long seed = -1, paths = -1;
    int lane_width = 4, threads = 1;
    double h = 3e-7, tolerance = 1e-6;

    static Run from_args(int argc, char** argv) {
        Run r;
        if (argc < 2) throw Usage("usage: lanetape_gpu price|gradcheck --config FILE [options]");
        r.command = argv[1];
        const bool gc = r.command == "gradcheck";
        if (!gc && r.command != "price") throw Usage("unknown command: " + r.command);
        std::map<std::string, std::function<void(const std::string&)>> set{
            {"--config", [&](const std::string& v) { r.config = v; }},
            {"--out-dir", [&](const std::string& v) { r.out_dir = v; }},
            {"--memory-mode", [&](const std::string& v) { r.memory_mode = v; }},
            {"--seed", [&](const std::string& v) { r.seed = std::stoll(v); }},
            {"--paths", [&](const std::string& v) { r.paths = std::stoll(v); }},
            {"--lane-width", [&](const std::string& v) { r.lane_width = std::stoi(v); }},
            {"--threads", [&](const std::string& v) { r.threads = std::stoi(v); }},
        };
        if (gc) {
            set["--fd-h"] = [&](const std::string& v) { r.h = std::stod(v); };
            set["--tolerance"] = [&](const std::string& v) { r.tolerance = std::stod(v); };
        }
        for (int i = 2; i < argc; i += 2) {
            auto it = set.find(argv[i]);
            if (it == set.end() || i + 1 >= argc)
                throw Usage(std::string("bad option: ") + argv[i]);
            try {
                it->second(argv[i + 1]);
            } catch (const std::logic_error&) {
                throw Usage(std::string("bad value for ") + argv[i] + ": " + argv[i + 1]);
            }
        }
        if (r.config.empty()) throw Usage("--config is required");
        if (r.memory_mode != "recompute" && r.memory_mode != "store")
            throw Usage("--memory-mode must be recompute or store");
        return r;
    }

    lanetape::ModelSpec model() const {
        if (!std::filesystem::exists(config)) throw Usage("no such config: " + config);
        lanetape::ModelSpec spec = lanetape::load_model_spec(config);
        if (paths >= 0) spec.mc.paths = static_cast<std::size_t>(paths);
        if (seed >= 0) spec.mc.seed = static_cast<std::uint64_t>(seed);
        return spec;
    }

    gpu::MCConfig mc(const lanetape::ModelSpec& spec) const {
        gpu::MCConfig c = gpu::mc_config(spec);
        c.lane_width = lane_width;
        c.worker_threads = threads;
        c.memory_mode = memory_mode == "store" ? gpu::MemoryMode::Store
                                               : gpu::MemoryMode::Recompute;
        return c;
    }

    void write(const char* file, const lanetape::ModelSpec& spec, const Json& results) const {
        Json doc;
        doc["config"] = Json{{"command", command},
                             {"model", lanetape::to_json(spec)},
                             {"run", Json{{"lane_width", lane_width},
                                          {"worker_threads", threads},
                                          {"memory_mode", memory_mode}}}};
        for (auto it = results.begin(); it != results.end(); ++it) doc[it.key()] = it.value();
        std::filesystem::create_directories(out_dir);
        const std::string path = (std::filesystem::path(out_dir) / file).string();
        std::ofstream(path) << doc.dump(2) << "\n";
        std::cout << "wrote " << path << "\n";
    }
};

void finite_or_throw(const std::vector<double>& v, const char* what) {
    for (double d : v)
        if (!std::isfinite(d)) throw gpu::EvalError(std::string(what) + " is not finite");
}

int price(const Run& run) {
    const lanetape::ModelSpec spec = run.model();
    gpu::Engine eng(gpu::to_gpu(spec));
    const auto res = eng.estimate_means(lanetape::pack_params(spec.heston, spec.grid), run.mc(spec));
    finite_or_throw(res.means, "price: means");
    run.write("price.json", spec,
              Json{{"means", res.means}, {"std_errors", res.std_errors}, {"paths", res.paths},
                   {"seed", spec.mc.seed}});
    for (std::size_t i = 0; i < res.means.size(); ++i)
        std::printf("E[y_%zu] = %.10g  (se %.3g)\n", i, res.means[i], res.std_errors[i]);
    return 0;
}

int gradcheck(const Run& run) {
    const lanetape::ModelSpec spec = run.model();
    gpu::Engine eng(gpu::to_gpu(spec));
    const gpu::MCConfig cfg = run.mc(spec);
    const std::vector<double> x = lanetape::pack_params(spec.heston, spec.grid);
    std::vector<double> targets = eng.estimate_means(x, cfg).means;
    finite_or_throw(targets, "gradcheck: means");
    for (double& t : targets) t *= 0.9;
    const gpu::GradientReport rep = eng.gradient_of_G(x, targets, cfg);
    finite_or_throw(rep.grad, "gradcheck: gradient");
    const std::vector<double> fd = eng.finite_diff_gradient_of_G(x, targets, cfg, run.h);
    finite_or_throw(fd, "gradcheck: finite differences");
    std::vector<double> rel;
    double worst = 0.0;
    for (std::size_t j = 0; j < fd.size(); ++j) {
        rel.push_back(std::fabs(rep.grad[j] - fd[j]) / std::fmax(std::fabs(rep.grad[j]), 1e-8));
        worst = std::fmax(worst, rel.back());
    }
    const bool ok = worst <= run.tolerance;
    run.write("gradcheck.json", spec,
              Json{{"h", run.h}, {"tolerance", run.tolerance}, {"max_rel_err", worst},
                   {"pass", ok}, {"G", rep.G}, {"grad", rep.grad}, {"fd_grad", fd},
                   {"rel_err", rel}});
    std::printf("adjoint vs central differences: max rel err %.3e (tolerance %g) %s\n", worst,
                run.tolerance, ok ? "PASS" : "FAIL");
    return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Run run = Run::from_args(argc, argv);
        return run.command == "price" ? price(run) : gradcheck(run);
    } catch (const gpu::EvalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
