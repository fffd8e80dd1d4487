/*
 * lanetape_b200.h — C ABI of the B200-native two-pass ∇G engine.
 *
 * This is the drop-in boundary for the hot path of arXiv 1901.04200 as the
 * reference `lanetape` library implements it. Every entry point names the
 * reference interface it replaces (paths relative to
 * /root/reference/proj/include/lanetape/):
 *
 *   ltg_gradient_of_G   <- lanetape::gradient_of_G(const Tape&, params, targets,
 *                          const MCConfig&)                 expectation.hpp:346-351
 *                          (and the Kernel/PathDrawSource overload :300-344)
 *   ltg_estimate_means  <- lanetape::estimate_means(const Tape&, params,
 *                          const MCConfig&)                 expectation.hpp:281-286
 *   ltg_finite_diff_gradient_of_G
 *                       <- lanetape::finite_diff_gradient_of_G   expectation.hpp:372-400
 *   ltg_gradient_of_G_draws / ltg_estimate_means_draws
 *                       <- the PathDrawSource overloads with BufferDrawSource /
 *                          SampleSpace draws  expectation.hpp:274-279, 287-294,
 *                          300-344, 354-367; rng.hpp:140-167
 *   ltg_fill_normals    <- lanetape::PhiloxNormalSource::fill    rng.hpp:113-127
 *   ltg_create_heston   <- lanetape::record_heston_program(ModelSpec) heston.hpp:327-329
 *                          (the GPU does not interpret tapes: the model description
 *                          itself is the program)
 *   ltg_pack_params     <- lanetape::pack_params                 heston.hpp:212-219
 *
 * Conventions (mirroring expectation.hpp / tape.hpp error behaviour):
 *   return LTG_OK (0) on success;
 *   LTG_EINVAL (1)   where the reference throws std::invalid_argument
 *                    (size mismatches, paths == 0, bad model, fresh_step2_paths
 *                    with store mode, ...);
 *   LTG_ENUMERIC (2) where the reference throws EvalError: the recorded
 *                    Heston program's sqrt(1 - rho^2) of a negative value
 *                    (heston.hpp:286, tape.hpp:261-263). Non-finite parameters
 *                    and non-finite results are NOT errors, as in the reference
 *                    library: the report carries the NaN / inf values (the
 *                    reference CLI's require_finite, tools/main.cpp, is the
 *                    caller's business; examples/lanetape_gpu exits 2 on them);
 *   LTG_ECUDA (3)    CUDA / NCCL runtime failure (no reference analogue);
 *   ltg_last_error(ctx) returns the message of the last failure on that
 *   context (ctx == NULL: last failure of a create call on this thread).
 * All host buffers are caller-owned. A context owns its device memory and
 * stream; one host thread may use a context at a time (the reference's
 * gradient_of_G is externally synchronous).
 *
 * There is no CPU fallback: every compute entry point runs CUDA kernels and
 * fails with LTG_ECUDA when no sm_100 device is usable.
 */
#ifndef LANETAPE_B200_H
#define LANETAPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTG_ABI_VERSION 3

#define LTG_OK 0
#define LTG_EINVAL 1
#define LTG_ENUMERIC 2
#define LTG_ECUDA 3

/* Instrument::Kind (heston.hpp:88-94) */
#define LTG_CALL 0
#define LTG_PUT 1

/* MemoryMode (expectation.hpp:17) — echoed into the report; the engine picks
 * its own device memory strategy (HBM checkpoints), see DESIGN.md §4. */
#define LTG_MODE_RECOMPUTE 0
#define LTG_MODE_STORE 1

/* arithmetic of the path simulation */
#define LTG_FP64 0
#define LTG_FP32 1

typedef struct ltg_ctx ltg_ctx;

/* ModelSpec minus McSettings.paths/seed (heston.hpp:96-114): HestonParams,
 * LeverageGrid, instruments, steps and dt. kappa..v0 and `leverage` are the
 * values the program is "recorded" at (pack_params order); the packed
 * parameter vector x passed to the compute calls overrides them. */
typedef struct ltg_heston_model {
    double mu;
    double s0;
    double kappa, theta, xi, rho, v0;
    const double* t_nodes;       /* n_t_nodes, strictly ascending */
    uint32_t n_t_nodes;
    const double* s_nodes;       /* n_s_nodes, strictly ascending */
    uint32_t n_s_nodes;
    const double* leverage;      /* n_t_nodes * n_s_nodes, t-major */
    const int32_t* inst_kind;    /* LTG_CALL / LTG_PUT */
    const double* inst_strike;
    const uint32_t* inst_maturity_step; /* in [1, steps] */
    uint32_t n_instruments;
    uint32_t steps;
    double dt;
} ltg_heston_model;

/* Correlated multi-asset log-Euler GBM (BASELINE config 4). Not a model of
 * the reference's model layer; its oracle is a program recorded with the
 * reference Tape API (oracle/ref_driver.cpp). Parameters are the n_assets
 * constant vols. Draw slot of (step k, asset a) is k*n_assets + a. */
typedef struct ltg_basket_model {
    uint32_t n_assets;           /* 1..16 */
    const double* s0;            /* n_assets */
    double r;                    /* drift constant */
    const double* chol;          /* n_assets*n_assets, lower-triangular, row-major */
    const double* sigma;         /* n_assets, recorded-at vols */
    const uint32_t* inst_asset;
    const int32_t* inst_kind;
    const double* inst_strike;
    const uint32_t* inst_maturity_step;
    uint32_t n_instruments;
    uint32_t steps;
    double dt;
} ltg_basket_model;

/* MCConfig (expectation.hpp:25-39). lane_width / worker_threads /
 * store_limit_bytes are CPU execution knobs with no GPU meaning and have no
 * field here (the C++ mirror, lanetape_b200.hpp, accepts and ignores them).
 * In particular the reference's store-mode budget check (expectation.hpp:
 * 307-319: std::invalid_argument when nodes x lanes x batches doubles exceed
 * store_limit_bytes) is NOT applied: memory_mode is echoed into the report
 * and the engine keeps its own device-memory plan (HBM checkpoints, the draw
 * store), which is bounded instead by ltg_set_hbm_budget. The reference's
 * other store-mode check, store + fresh_step2_paths -> invalid, is kept.
 * precision = LTG_FP32 (config 5's variant): Heston-SLV programs only;
 * gradients additionally need the Feller condition 2*kappa*theta >= xi^2 of
 * the parameters passed (LTG_EINVAL otherwise; DESIGN.md §6 states the
 * per-config accuracy bars). */
typedef struct ltg_mc_config {
    uint64_t paths;
    uint64_t seed;
    int32_t antithetic;
    int32_t fresh_step2_paths;
    int32_t memory_mode;         /* LTG_MODE_*, echoed */
    int32_t precision;           /* LTG_FP64 / LTG_FP32 */
} ltg_mc_config;

/* GradientReport (expectation.hpp:62-82). Array members are caller-owned
 * output buffers; std_errors may be NULL. */
typedef struct ltg_report {
    double G;
    double* means;               /* m */
    double* lambda;              /* m */
    double* grad;                /* M */
    double* std_errors;          /* m, optional */
    uint64_t paths;
    uint64_t seed;
    int32_t mode;
} ltg_report;

/* Device timings of the last compute call on a context (CUDA events on the
 * context stream). */
typedef struct ltg_timing {
    double pass1_ms;             /* forward kernel(s) */
    double pass2_ms;             /* adjoint kernel(s) */
    double reduce_ms;            /* chunk reductions + finalisation + collectives */
    double total_ms;
    uint64_t paths_pass1;
    uint64_t paths_pass2;
    uint32_t launches;           /* kernels this library launched in the call */
    uint32_t seg_steps;          /* checkpoint interval used (Heston), 0 if none */
    uint64_t ckpt_bytes;         /* HBM checkpoint / store table written by pass 1 */
    uint64_t z_bytes;            /* HBM draw store written by pass 1 (read by pass 2) */
    uint32_t safe_rerun;         /* 1: a fast kernel flagged an out-of-range argument and
                                    the call was redone with the exact slow paths */
    uint32_t graph;              /* 0: the call's work was enqueued eagerly; 1: captured into
                                    a CUDA graph (second call of its shape); 2: replayed from
                                    that graph (single-GPU contexts; LTG_GRAPH=0 disables) */
} ltg_timing;

/* Path sharding plan: the path set is cut into fixed chunks whose size
 * depends only on the total path count, so chunk partial sums and their
 * ascending-order reduction are bitwise independent of the rank count. */
typedef struct ltg_shard {
    uint64_t chunk_paths;
    uint64_t n_chunks;
    uint64_t chunk_begin;        /* this rank's [chunk_begin, chunk_end) */
    uint64_t chunk_end;
    uint64_t path_begin;         /* [path_begin, path_end) of the global path index space */
    uint64_t path_end;
} ltg_shard;

int ltg_abi_version(void);

int ltg_create_heston(const ltg_heston_model* model, int device, ltg_ctx** out);
int ltg_create_basket(const ltg_basket_model* model, int device, ltg_ctx** out);
/* Single-process multi-GPU context (the reference's host is one process):
 * one member context per listed device, NCCL communicators from
 * ncclCommInitAll, member i = rank i. Every compute call then runs on all
 * devices concurrently (one host thread each), sharded and reduced exactly as
 * ltg_attach_nccl's one-process-per-GPU mode — the same bits for any device
 * count. Single-device diagnostics (fill_normals, inverse_normal,
 * path_payoffs, chunk_sums) run on the first device. */
int ltg_create_heston_devices(const ltg_heston_model* model, const int* devices, int n,
                              ltg_ctx** out);
int ltg_create_basket_devices(const ltg_basket_model* model, const int* devices, int n,
                              ltg_ctx** out);
void ltg_destroy(ltg_ctx* ctx);
const char* ltg_last_error(const ltg_ctx* ctx);

size_t ltg_num_params(const ltg_ctx* ctx);   /* M */
size_t ltg_num_outputs(const ltg_ctx* ctx);  /* m */
size_t ltg_num_randoms(const ltg_ctx* ctx);  /* N per path */
int ltg_pack_params(const ltg_ctx* ctx, double* x, size_t M);

int ltg_gradient_of_G(ltg_ctx* ctx, const double* x, size_t M, const double* targets, size_t m,
                      const ltg_mc_config* cfg, ltg_report* report);
/* The same report as ltg_gradient_of_G, with pass 2 replaced by pathwise
 * tangents (forward mode): ∇G is linear in λ, so one forward sweep that
 * carries d(log S)/dx and dV/dx for every parameter gives, per instrument i,
 * J_i = Σ_p ∂y_i/∂x and then grad = Σ_i λ_i J_i / P — the reference's
 * estimator on the same paths, same derivative conventions, different
 * summation order (agrees with ltg_gradient_of_G to ~1e-14). Cheaper than the
 * adjoint when M is small: fp64 Heston models with one leverage column and at
 * most 4 leverage rows (M = 5 + rows <= 9); LTG_EINVAL otherwise. Not a
 * reference interface: an engine alternative to expectation.hpp:300-351. */
int ltg_gradient_of_G_tangent(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                              size_t m, const ltg_mc_config* cfg, ltg_report* report);
int ltg_estimate_means(ltg_ctx* ctx, const double* x, size_t M, const ltg_mc_config* cfg,
                       double* means, double* std_errors);
int ltg_finite_diff_gradient_of_G(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                                  size_t m, const ltg_mc_config* cfg, double h, double* grad);

/* Caller-supplied draws: the reference's PathDrawSource overloads with a
 * materialised source — BufferDrawSource (rng.hpp:140-167; also what
 * BufferDrawSource::materialize makes of any user PathDrawSource) and
 * SampleSpace (expectation.hpp:46-54, 85-101). Row p (dim doubles) holds the
 * draws of path p, in the program's slot order (Heston: slot 2k drives V,
 * 2k+1 the independent part of S; basket: slot k*n_assets + a). */
typedef struct ltg_draws {
    const double* data;          /* rows * dim, path-major, caller-owned */
    uint64_t rows;
    uint64_t dim;                /* must equal ltg_num_randoms (else LTG_EINVAL) */
} ltg_draws;

/* gradient_of_G(kernel, params, targets, src, cfg)   expectation.hpp:300-344
 * with src = the caller's draws: pass 1 reads rows [0, paths), pass 2 the same
 * rows, or rows [paths, 2*paths) with fresh_step2_paths. cfg->seed is only
 * echoed into the report and cfg->antithetic is unused (the source fixes the
 * draws), as in the reference. Too few rows -> LTG_EINVAL (the reference's
 * std::out_of_range from fill). The SampleSpace overload (:354-367) is this
 * call with rows = paths = scenarios, seed 0, recompute mode. */
int ltg_gradient_of_G_draws(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                            size_t m, const ltg_draws* src, const ltg_mc_config* cfg,
                            ltg_report* report);
/* estimate_means(kernel, params, src, paths, workers)  expectation.hpp:274-279
 * (and the SampleSpace overload :287-294 with paths = scenarios); fp64. */
int ltg_estimate_means_draws(ltg_ctx* ctx, const double* x, size_t M, const ltg_draws* src,
                             uint64_t paths, double* means, double* std_errors);

/* One chunk of the two passes, unreduced (SURVEY §8(c) per-chunk parity):
 * over the global paths [path0, path0+npaths) of PhiloxNormalSource(seed),
 * the pass-1 sums Σy, Σy² (detail::forward_pass, expectation.hpp:152-198) and
 * the pass-2 parameter-adjoint total seeded with the caller's lambda
 * (detail::reverse_pass, :204-249) — the totals before the division by P.
 * sums/sumsq: m, adjoint: M. Diagnostic / parity entry point. */
int ltg_chunk_sums(ltg_ctx* ctx, const double* x, size_t M, const double* lambda, size_t m,
                   uint64_t seed, int antithetic, uint64_t path0, uint64_t npaths,
                   double* sums, double* sumsq, double* adjoint);

/* PhiloxNormalSource(seed, dim, antithetic).fill(path) for paths
 * [path0, path0+npaths), generated on the GPU; out is npaths*dim, path-major. */
int ltg_fill_normals(ltg_ctx* ctx, uint64_t seed, size_t dim, int antithetic, uint64_t path0,
                     uint64_t npaths, double* out);

/* inverse_normal_cdf (rng.hpp:45-85) of n uniforms p[i] through the device
 * AS241 (central and both tail rows; the path kernels run the same code fused
 * with Philox). p must lie in (0,1) (LTG_EINVAL otherwise, where the reference
 * throws) and be of the generator's form (2k+1)*2^-53, which makes q = p - 0.5
 * exact as in the reference. Diagnostic / parity entry point. */
int ltg_inverse_normal(ltg_ctx* ctx, const double* p, size_t n, double* z);

/* Per-path outputs of the program (forward_eval, tape.hpp:276-331, on the
 * draws PhiloxNormalSource(seed).fill(p)) for p in [path0, path0+npaths):
 * y is npaths*m, path-major. */
int ltg_path_payoffs(ltg_ctx* ctx, const double* x, size_t M, uint64_t seed, int antithetic,
                     uint64_t path0, uint64_t npaths, double* y);

int ltg_last_timing(const ltg_ctx* ctx, ltg_timing* out);

/* Device timing of calls (ltg_last_timing's pass1_ms / pass2_ms / reduce_ms /
 * total_ms): on (1, the default) records CUDA events around the passes; off
 * (0) records none, and those fields read 0. Events cost a small call (or a
 * replayed graph, whose event-record nodes they become) ~10 us of its ~70,
 * so latency-bound callers (a calibration loop) switch them off. Results do
 * not depend on it. */
int ltg_set_timing(ltg_ctx* ctx, int on);

/* Cap (bytes, per GPU) of the HBM the context may hold for its checkpoint
 * table and draw store; 0 (the default) uses the free device memory minus a
 * 2 GiB reserve. Results do not depend on it, only the speed of pass 2. */
int ltg_set_hbm_budget(ltg_ctx* ctx, uint64_t bytes);

/* 1 when the GPU inverse-normal uses a log() validated bit-for-bit against
 * this host's libm (the reference's random stream is reproduced exactly);
 * 0 when that check failed and the GPU fell back to CUDA's log(). */
int ltg_rng_exact(const ltg_ctx* ctx);

/* Multi-GPU (one process per GPU). Pure host arithmetic, no device use. */
int ltg_shard_plan(uint64_t paths, int rank, int world, ltg_shard* out);
/* NCCL is loaded at run time (the libnccl.so.2 already in the process, e.g.
 * torch's, else the system one). Rank 0 creates the id, the caller
 * broadcasts it, every rank attaches. After attach, compute calls shard the
 * path set by ltg_shard_plan and all-gather chunk partials over NCCL; every
 * rank returns the identical report. */
int ltg_nccl_unique_id(unsigned char id[128]);
int ltg_attach_nccl(ltg_ctx* ctx, const unsigned char id[128], int rank, int world);

/* Diagnostic: measured FP64 issue rate of `device` — thread-level FP64
 * instructions per second, the fastest of DFMA, DMUL+DADD and DADD streams
 * (8 independent chains per thread, full occupancy, best of 3) — the
 * roofline denominator reported by bench.py. */
int ltg_probe_fp64_rate(int device, double* fp64_per_s, double* sm_clock_hz);
/* Diagnostic: measured FP32 FFMA issue rate (thread instructions per second,
 * 8 chains per thread, full occupancy) — the fp32 mode's roofline denominator. */
int ltg_probe_fp32_rate(int device, double* fp32_per_s);

/* Host-only self-test of the random stream's log(): locates and validates
 * the host libm table (as context creation does) and compares the GPU's
 * restated log sequence, evaluated on the host, with log() on n tail
 * arguments. Returns 0 when a table was found; *mismatches counts
 * disagreements (expected 0), *exact is what ltg_rng_exact would report. */
int ltg_rng_selftest(uint64_t n, uint64_t* mismatches, int* exact);

#ifdef __cplusplus
}
#endif

#endif /* LANETAPE_B200_H */
