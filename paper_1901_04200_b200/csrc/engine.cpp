// engine.cpp — host side of the C ABI (include/lanetape_b200.h).
//
// Orchestrates gradient_of_G (expectation.hpp:300-344) on one GPU or on one
// rank of a multi-GPU job:
//   pass 1  forward kernel over this rank's chunks      -> chunk partials, HBM checkpoints
//   [NCCL all-gather of chunk partial rows]
//   fixed-order chunk reduction -> means, std errors, lambda, G   (all on device)
//   pass 2  adjoint kernel over the same chunks          -> chunk partials
//   [NCCL all-gather]  fixed-order reduction -> grad = total / P
//   one device->host copy of {G, means, se, lambda, grad} and the rare flag
// The fast kernels flag arguments outside their exact range; a flagged call
// (flag all-reduced over ranks) is rerun with the SAFE kernels, bit-identical
// where both are defined. ltg_gradient_of_G_tangent replaces pass 2 by the
// pathwise-tangent kernel (run_tangent); ltg_chunk_sums runs one global path
// range of both passes unreduced (parity checks).
// Validation mirrors the reference's std::invalid_argument sites (LTG_EINVAL)
// and its EvalError site (LTG_ENUMERIC); non-finite results are returned, as
// the reference library returns them.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <condition_variable>
#include <functional>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lanetape_b200.h"
#include "kernels.h"

namespace ltg {
std::string discover_glibc_math(RngConsts& K, RngTables& T);
void fill_as241(RngConsts& K);
}  // namespace ltg

using namespace ltg;

namespace {

thread_local std::string g_create_error;

struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Failure(LTG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cuda_check(cudaMalloc(&p, b), "cudaMalloc");
        bytes = b;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ---- NCCL, resolved at run time ----
struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    std::mutex mu;

    bool load(std::string& why) {
        std::lock_guard<std::mutex> lock(mu);  // contexts may attach from several threads
        if (lib) return true;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return false;
        }
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(dlsym(lib, "ncclCommInitRank"));
        CommInitAll = reinterpret_cast<decltype(CommInitAll)>(dlsym(lib, "ncclCommInitAll"));
        AllGather = reinterpret_cast<decltype(AllGather)>(dlsym(lib, "ncclAllGather"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(dlsym(lib, "ncclAllReduce"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(dlsym(lib, "ncclCommDestroy"));
        GetErrorString =
            reinterpret_cast<decltype(GetErrorString)>(dlsym(lib, "ncclGetErrorString"));
        if (!GetUniqueId || !CommInitRank || !CommInitAll || !AllGather || !AllReduce ||
            !CommDestroy || !GetErrorString) {
            why = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
Nccl& nccl() {
    static Nccl n;
    return n;
}

ltg_shard make_plan(uint64_t paths, int rank, int world) {
    ltg_shard s{};
    // chunk size depends on the total path count only
    uint64_t r = paths / (uint64_t(8192) * kBlock);
    uint64_t R = 1;
    while (R * 2 <= r && R < 8) R *= 2;
    s.chunk_paths = uint64_t(kBlock) * R;
    s.n_chunks = (paths + s.chunk_paths - 1) / s.chunk_paths;
    const uint64_t per = (s.n_chunks + world - 1) / world;  // padded equal split for all-gather
    s.chunk_begin = std::min<uint64_t>(per * rank, s.n_chunks);
    s.chunk_end = std::min<uint64_t>(per * (rank + 1), s.n_chunks);
    s.path_begin = std::min<uint64_t>(s.chunk_begin * s.chunk_paths, paths);
    s.path_end = std::min<uint64_t>(s.chunk_end * s.chunk_paths, paths);
    return s;
}

// Per-context call block (d_res): the report a call copies back in one D2H
// copy, followed by the call's flag words, cleared by one memset:
//   [G | means m | std_errors m | lambda m | grad M] doubles, then
//   uint32 flags[16]: flags[0] the fast arithmetic's out-of-range flag,
//   flags[1 + s] the dynamic chunk scheduler of launch slot s (0-2)
constexpr int kFlagWords = 16;

uint64_t chunks_per_rank(const ltg_shard& s, int world) {
    return (s.n_chunks + world - 1) / world;
}

}  // namespace

// Test-only in-process collective for member contexts that share one GPU
// (LTG_LOOPBACK=1 with ltg_create_*_devices): the exchanges NCCL performs,
// done with device-to-device copies between the members' tables and a host
// barrier, so the multi-rank code paths (shard plans, per-rank rows, the
// all-gather layout, the rare-flag reduction) run for real on one GPU.
struct Loopback {
    explicit Loopback(int w) : world(w), tables(w, nullptr), flags(w, 0) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<double*> tables;
    std::vector<uint32_t> flags;
    void barrier() {
        std::unique_lock<std::mutex> lock(mu);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lock, [&] { return generation != gen; });
        }
    }
};

namespace ltg {
thread_local LaunchHook* t_launch_hook = nullptr;
}

// CUDA-graph replay of a call on a single-GPU context (run_body). A call's
// device work — the H2D copy of x and the targets, the counter memsets, the
// pass kernels, the reductions, the timing events and the D2H copies of the
// report and the rare flag — is captured into a graph the second time a call
// of the same shape arrives; later calls of that shape replay it with one
// cudaGraphLaunch. The host code of the call still runs, with the hook
// installed in Update mode: every enqueue is compared with the captured
// sequence, kernels whose arguments changed (parameters, seed, ...) get their
// graph node updated (cudaGraphExecKernelNodeSetParams), and any other
// difference (a buffer moved, a different plan) drops the graph and runs the
// call eagerly.
struct GraphRec : LaunchHook {
    enum Mode { Capture, Update } mode = Capture;
    struct Kernel {
        const void* func;
        dim3 grid, block;
        size_t smem;
        std::vector<size_t> sizes;
        std::vector<char> args;
    };
    struct Op {  // memset / copy / event: kind and operands must repeat exactly
        int kind;
        const void* a;
        const void* b;
        size_t n;
    };
    std::vector<Kernel> kernels;
    std::vector<Op> ops;
    std::vector<cudaGraphNode_t> knodes;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::string key;
    size_t kcur = 0, ocur = 0;
    bool mismatch = false;

    ~GraphRec() override { reset(); }
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        kernels.clear();
        ops.clear();
        knodes.clear();
        key.clear();
    }
    static bool same(dim3 a, dim3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
    cudaError_t launch(const void* func, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       void** args, const size_t* sizes, int n) override {
        std::vector<size_t> sz(sizes, sizes + n);
        std::vector<char> bytes;
        for (int i = 0; i < n; ++i)
            bytes.insert(bytes.end(), static_cast<char*>(args[i]), static_cast<char*>(args[i]) + sizes[i]);
        if (mode == Capture) {
            kernels.push_back({func, grid, block, smem, sz, bytes});
            return cudaLaunchKernel(func, grid, block, args, smem, st);
        }
        if (kcur >= kernels.size()) {
            mismatch = true;
            return cudaSuccess;
        }
        Kernel& k = kernels[kcur++];
        if (k.func != func || !same(k.grid, grid) || !same(k.block, block) || k.smem != smem ||
            k.sizes != sz) {
            if (std::getenv("LTG_GRAPH_DEBUG"))
                std::fprintf(stderr, "graph: kernel %zu differs (func %d grid %d smem %d)\n",
                             kcur - 1, k.func != func, !same(k.grid, grid), k.smem != smem);
            mismatch = true;
            return cudaSuccess;
        }
        if (k.args != bytes && !mismatch) {
            cudaKernelNodeParams p{};
            p.func = const_cast<void*>(func);
            p.gridDim = grid;
            p.blockDim = block;
            p.sharedMemBytes = (unsigned)smem;
            p.kernelParams = args;
            const cudaError_t e = cudaGraphExecKernelNodeSetParams(exec, knodes[kcur - 1], &p);
            if (e != cudaSuccess) {
                if (std::getenv("LTG_GRAPH_DEBUG"))
                    std::fprintf(stderr, "graph: kernel node %zu update failed: %s\n", kcur - 1,
                                 cudaGetErrorString(e));
                mismatch = true;
                cudaGetLastError();
                return cudaSuccess;
            }
            k.args.swap(bytes);
        }
        return cudaSuccess;
    }
    // non-kernel enqueue: true = enqueue it (eager / capture), false = the graph has it
    bool op(int kind, const void* a, const void* b, size_t n) {
        if (mode == Capture) {
            ops.push_back({kind, a, b, n});
            return true;
        }
        if (ocur >= ops.size() || ops[ocur].kind != kind || ops[ocur].a != a || ops[ocur].b != b ||
            ops[ocur].n != n) {
            if (std::getenv("LTG_GRAPH_DEBUG"))
                std::fprintf(stderr, "graph: op %zu (kind %d, %zu bytes) differs\n", ocur, kind, n);
            mismatch = true;
        }
        ++ocur;
        return false;
    }
};
thread_local GraphRec* t_rec = nullptr;

// persistent worker threads of a multi-device context (group_run): member i
// > 0 runs on worker i - 1, member 0 on the calling thread
struct Pool {
    std::vector<std::thread> threads;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::function<void(size_t)> job;
    uint64_t gen = 0;
    size_t pending = 0;
    bool stop = false;
    explicit Pool(size_t workers) {
        for (size_t i = 0; i < workers; ++i)
            threads.emplace_back([this, i] {
                uint64_t seen = 0;
                for (;;) {
                    std::function<void(size_t)> fn;
                    {
                        std::unique_lock<std::mutex> lock(mu);
                        cv.wait(lock, [&] { return stop || gen != seen; });
                        if (stop) return;
                        seen = gen;
                        fn = job;
                    }
                    fn(i + 1);
                    std::lock_guard<std::mutex> lock(mu);
                    if (--pending == 0) done_cv.notify_all();
                }
            });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lock(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : threads) t.join();
    }
    // fn(0) on the caller, fn(1..workers) on the workers; returns when all are done
    void run(const std::function<void(size_t)>& fn) {
        {
            std::lock_guard<std::mutex> lock(mu);
            job = fn;
            pending = threads.size();
            ++gen;
        }
        cv.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lock(mu);
        done_cv.wait(lock, [&] { return pending == 0; });
    }
};

struct ltg_ctx {
    // single-process multi-GPU context (ltg_create_*_devices): one member
    // context per device, member i = NCCL rank i; the group itself has no
    // device state and runs every call on all members concurrently
    std::vector<std::unique_ptr<ltg_ctx>> members;
    std::unique_ptr<Pool> pool;      // the members' host threads (members.size() - 1 workers)
    std::shared_ptr<Loopback> loop;  // test-only collective instead of NCCL (see Loopback)
    // call graphs by call shape (run_body): seen once -> captured on the
    // next call -> replayed; a few shapes (gradient / means / tangent calls
    // of a calibration loop) are kept
    std::map<std::string, std::unique_ptr<GraphRec>> graphs;
    std::vector<std::string> graph_order;  // insertion order, oldest first
    uint64_t hbm_budget = 0;         // ltg_set_hbm_budget: cap of checkpoints + draws (0: free HBM)
    int kind = 0;  // 0 Heston SLV, 1 basket
    uint64_t path_base = 0;  // global index of path 0 of a call (ltg_chunk_sums; else 0)
    bool ready = false;  // device state initialised
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[8] = {};
    // ev_at[i]: the event that marks timing point i of the last call — its own,
    // or an earlier one recorded at the same point of the stream (same_event),
    // so a replayed graph carries no back-to-back event nodes
    int ev_at[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    std::string err;
    std::string rng_note;

    // model (host)
    uint32_t steps = 0, cols = 1, rows = 1, nlev = 1, m = 0, M = 0, N = 0;
    double s0 = 0, mu = 0, dt = 0;
    std::vector<double> x0;
    std::vector<double> h_x;  // parameters of the current call
    // [x | targets] on the device (d_x) when they do not fit the kernels'
    // by-value arguments (upload_x), else null
    const double* x_src = nullptr;
    std::vector<double> h_t;  // targets of the current call (empty: none)
    // lean calls: the host buffer the call's last reduction publishes the
    // report into (Finish::pub), null otherwise; flag_clean: the rare flag is
    // known to be zero (the last lean call's final kernel cleared it)
    double* pub = nullptr;
    bool flag_clean = true;
    std::vector<MaturityEvent> events;
    std::vector<uint32_t> inst_order;

    // basket model (host)
    uint32_t n_assets = 0;
    double r = 0;
    std::vector<double> chol, s0v;
    bool store_ok = false;  // pass 1 of the current call wrote the basket store

    // model (device)
    DevBuf d_snodes, d_rowoff, d_events, d_order, d_strike, d_kind, d_asset, d_tab;
    RngConsts h_rc{};
    RngTables h_tab{};
    uint32_t seg_steps = 16;  // checkpoint interval of the current call
    int fp32 = 0;             // precision of the current call (Heston only)
    int safe = 0;             // 1: exact slow paths for every argument (heston_step SAFE)

    // per-call buffers
    DevBuf d_x, d_part1, d_part2, d_groups, d_tot1, d_tot2, d_res,
        d_ckpt, d_ztab, d_normals;
    uint64_t z_chunks = 0;  // leading local chunks whose draws pass 1 stored
    // caller-supplied draws of the current *_draws call (DrawScope): rows
    // [row0A, row0A + rowsA) of the caller's buffer for pass 1, then, with
    // fresh_step2_paths, rows [row0B, row0B + rowsA) for pass 2
    DevBuf d_draws;
    bool draws_on = false;
    uint64_t draws_rowsA = 0, draws_row0A = 0, draws_row0B = 0;
    // inputs and outcome of the last HBM plan (run_pass1); a call with the
    // same inputs reuses it without querying the device (its buffers are held)
    std::string plan_key;
    uint32_t plan_ks = 16;
    uint64_t plan_z = 0;
    bool plan_chosen = false;
    double* h_stage = nullptr;  // pinned
    size_t h_stage_bytes = 0;

    // multi-GPU
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    int timing_pending = 0;    // 1 / 2: `timing`'s device times still to read (settle_timing)
    bool timing_on = true;     // ltg_set_timing

    ltg_timing timing{};

    ~ltg_ctx() {
        if (comm) nccl().CommDestroy(comm);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
        if (h_stage) cudaFreeHost(h_stage);
    }

    double* stage(size_t doubles) {
        if (doubles * 8 > h_stage_bytes) {
            if (h_stage) cudaFreeHost(h_stage);
            h_stage = nullptr;
            cuda_check(cudaMallocHost(&h_stage, doubles * 8), "cudaMallocHost");
            h_stage_bytes = doubles * 8;
        }
        return h_stage;
    }
};

namespace {

size_t out_doubles(const ltg_ctx* c) { return 1 + 3 * size_t(c->m) + c->M; }
double* res_ptr(ltg_ctx* c) { return c->d_res.as<double>(); }
double* grad_ptr(ltg_ctx* c) { return c->d_res.as<double>() + 1 + 3 * size_t(c->m); }
uint32_t* flags_ptr(ltg_ctx* c) {
    return reinterpret_cast<uint32_t*>(c->d_res.as<double>() + out_doubles(c));
}
uint32_t* rare_ptr(ltg_ctx* c) { return flags_ptr(c); }
uint32_t* counter_ptr(ltg_ctx* c, int slot) { return flags_ptr(c) + 1 + slot; }
// the call block, allocated once the model's sizes are known (create)
void alloc_call_block(ltg_ctx* c) {
    c->d_res.ensure(out_doubles(c) * 8 + kFlagWords * 4);
    cuda_check(cudaMemset(c->d_res.p, 0, c->d_res.bytes), "memset");
}

template <typename Fn>
int guarded(ltg_ctx* ctx, Fn&& fn) {
    try {
        if (ctx && ctx->ready) cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        fn();
        return LTG_OK;
    } catch (const Failure& f) {
        if (ctx) ctx->err = f.what();
        return f.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return LTG_ECUDA;
    }
}

// validation: a literal message costs nothing on success; composed messages
// go through require_f, which builds them only on failure (a small call's
// host path runs a dozen checks)
void require(bool ok, const char* msg) {
    if (!ok) throw Failure(LTG_EINVAL, msg);
}
void require(bool ok, const std::string& msg) {  // (context creation)
    if (!ok) throw Failure(LTG_EINVAL, msg);
}
template <typename Msg>
void require_f(bool ok, Msg&& msg) {
    if (!ok) throw Failure(LTG_EINVAL, msg());
}

bool is_group(const ltg_ctx* c) { return c && !c->members.empty(); }

// Run fn(member, index) on every member of a multi-GPU context, one host
// thread per device (their NCCL collectives meet; the threads persist with
// the context), and report the first failure. Validation failures happen identically on every member before any
// collective, so a bad argument cannot leave some members waiting.
void settle_timing(ltg_ctx* c);
void set_pub(ltg_ctx* c, Finish& fin);
void set_targets(ltg_ctx* c, Finish& fin);

// Work::fuse: the launch's last CTA reduces its chunk table and finishes the
// call (finish.cuh fused_tail) instead of launch_reduce_chunks — for tables
// small enough that one CTA's (group, column) items cover them in at most
// two rounds, and only on one GPU without a collective (its rows need no
// all-gather first), with the fast Philox kernels (a safe rerun or caller
// draws reduce separately). LTG_FUSE_REDUCE=0 turns it off (tests: both forms).
bool fuse_reduce(ltg_ctx* c, Work& w, uint32_t width, double* tot, const Finish& fin) {
    static const bool on = [] {
        const char* e = std::getenv("LTG_FUSE_REDUCE");
        return !(e && e[0] == '0');
    }();
    const uint64_t ng = (w.n_chunks + kGroup - 1) / kGroup;
    if (!on || c->world != 1 || c->comm || c->loop || c->safe || c->draws_on || w.n_chunks == 0 ||
        w.chunk_begin != 0 || ng * width > 2 * uint64_t(kBlock))
        return false;
    w.fuse = 1;
    w.done = counter_ptr(c, 3);
    w.groups = c->d_groups.as<double>();
    w.tot = tot;
    w.fin = fin;
    return true;
}

template <typename Fn>
int group_run(ltg_ctx* g, Fn&& fn) {
    const size_t n = g->members.size();
    std::vector<int> rc(n, LTG_OK);
    if (!g->pool) g->pool = std::make_unique<Pool>(n - 1);
    g->pool->run([&](size_t i) { rc[i] = fn(g->members[i].get(), i); });
    for (size_t i = 0; i < n; ++i)
        if (rc[i] != LTG_OK) {
            g->err = g->members[i]->err;
            return rc[i];
        }
    for (const auto& m : g->members) {
        cudaSetDevice(m->device);
        settle_timing(m.get());
    }
    g->timing = g->members[0]->timing;  // with the slowest member's total
    for (const auto& m : g->members)
        g->timing.total_ms = std::max(g->timing.total_ms, m->timing.total_ms);
    return LTG_OK;
}

// A single-device diagnostic (draws, per-path outputs, chunk sums) on member
// 0, its communicator detached for the call.
template <typename Fn>
int group_solo(ltg_ctx* g, Fn&& fn) {
    ltg_ctx* m = g->members[0].get();
    const ncclComm_t comm = m->comm;
    const std::shared_ptr<Loopback> loop = m->loop;
    const int rank = m->rank, world = m->world;
    m->comm = nullptr;
    m->loop = nullptr;
    m->rank = 0;
    m->world = 1;
    const int rc = fn(m);
    m->comm = comm;
    m->loop = loop;
    m->rank = rank;
    m->world = world;
    if (rc != LTG_OK) g->err = m->err;
    g->timing = m->timing;
    return rc;
}

template <typename T>
void upload(DevBuf& b, const std::vector<T>& v) {
    b.ensure(std::max<size_t>(1, v.size()) * sizeof(T));
    if (!v.empty())
        cuda_check(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
                   "upload");
}

void init_common(ltg_ctx* c, int device) {
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    require(device >= 0 && device < n, "device index out of range");
    c->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        throw Failure(LTG_ECUDA, std::string("device ") + prop.name +
                                     " is not sm_100 (this library is built for sm_100a only)");
    cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    for (auto& e : c->ev) cuda_check(cudaEventCreate(&e), "event");
    fill_as241(c->h_rc);
    c->rng_note = discover_glibc_math(c->h_rc, c->h_tab);
    for (int k = 0; k < 8; ++k) c->h_tab.as241_far[k] = make_double2(c->h_rc.num[2][k], c->h_rc.den[2][k]);
    c->d_tab.ensure(sizeof(RngTables));
    cuda_check(cudaMemcpy(c->d_tab.p, &c->h_tab, sizeof(RngTables), cudaMemcpyHostToDevice),
               "rng upload");
    c->ready = true;
}

// maturity events from instrument maturity steps (stable order, like the
// HestonSimulator bucketing, heston.hpp:336-375)
void build_events(ltg_ctx* c, const std::vector<uint32_t>& mats) {
    std::vector<uint32_t> order(mats.size());
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return mats[a] < mats[b]; });
    c->events.clear();
    for (uint32_t i = 0; i < order.size(); ++i) {
        const uint32_t st = mats[order[i]];
        if (c->events.empty() || c->events.back().step != st)
            c->events.push_back(MaturityEvent{st, i, i + 1});
        else
            c->events.back().end = i + 1;
    }
    c->inst_order = order;
    upload(c->d_events, c->events);
    upload(c->d_order, c->inst_order);
}

size_t floor_index(const std::vector<double>& nodes, double x) {
    auto it = std::upper_bound(nodes.begin(), nodes.end(), x);
    return it == nodes.begin() ? 0 : size_t(it - nodes.begin() - 1);
}

void all_gather_rows(ltg_ctx* c, double* table, uint64_t per_rank, uint32_t width) {
    if (c->loop) {
        Loopback& L = *c->loop;
        const size_t count = size_t(per_rank) * width;
        cuda_check(cudaStreamSynchronize(c->stream), "synchronize");  // own rows written
        L.tables[c->rank] = table;
        L.barrier();  // every member's rows are written
        for (int r = 0; r < L.world; ++r)
            if (r != c->rank)
                cuda_check(cudaMemcpyAsync(table + size_t(r) * count, L.tables[r] + size_t(r) * count,
                                           count * 8, cudaMemcpyDeviceToDevice, c->stream),
                           "loopback all-gather");
        cuda_check(cudaStreamSynchronize(c->stream), "synchronize");
        L.barrier();  // no member reuses its table before every copy is done
        return;
    }
    if (!c->comm) return;  // (an attached single-rank comm still runs the collective)
    const size_t count = size_t(per_rank) * width;
    const ncclResult_t r = nccl().AllGather(table + size_t(c->rank) * count, table, count,
                                            ncclFloat64, c->comm, c->stream);
    if (r != ncclSuccess)
        throw Failure(LTG_ECUDA, std::string("ncclAllGather: ") + nccl().GetErrorString(r));
}

// Basket step constants from the parameters, rounded exactly as the recorded
// program computes them (oracle/ref_driver.cpp record_basket).
BasketArgs basket_args(ltg_ctx* c, const double* x) {
    BasketArgs a{};
    a.n = c->n_assets;
    a.steps = c->steps;
    a.m = c->m;
    a.n_events = (uint32_t)c->events.size();
    a.dt = c->dt;
    volatile double sq = std::sqrt(c->dt);
    a.sqdt = sq;
    for (uint32_t i = 0; i < a.n; ++i) {
        for (uint32_t j = 0; j < a.n; ++j) a.chol[i * kMaxAssets + j] = c->chol[i * a.n + j];
        a.s0[i] = c->s0v[i];
        a.sigma[i] = x[i];
        volatile double ss = x[i] * x[i];
        volatile double hs = 0.5 * ss;
        volatile double rd = c->r - hs;
        a.drift[i] = rd * c->dt;
        a.vol[i] = x[i] * a.sqdt;
    }
    a.events = c->d_events.as<MaturityEvent>();
    a.inst_order = c->d_order.as<uint32_t>();
    a.asset = c->d_asset.as<uint32_t>();
    a.strike = c->d_strike.as<double>();
    a.kind = c->d_kind.as<int32_t>();
    a.tables = c->d_tab.as<RngTables>();
    a.rc = c->h_rc;
    a.safe = c->safe;
    a.rare = rare_ptr(c);
    if (c->draws_on) {
        a.draws = c->d_draws.as<double>();
        a.draws_row0 = c->draws_row0A;
    }
    return a;
}

HestonArgs heston_args(ltg_ctx* c, const double* x) {
    HestonArgs a{};
    a.steps = c->steps;
    a.cols = c->cols;
    a.rows = c->rows;
    a.nlev = c->nlev;
    a.m = c->m;
    a.n_events = (uint32_t)c->events.size();
    a.s0 = c->s0;
    a.dt = c->dt;
    a.sqdt = std::sqrt(c->dt);
    a.mu_dt = c->mu * c->dt;
    a.half_dt = 0.5 * c->dt;
    // step constants, rounded exactly as the reference tape computes them
    a.sc.kappa = x[0];
    a.sc.theta = x[1];
    a.sc.xi = x[2];
    a.sc.rho = x[3];
    {
        volatile double rr = x[3] * x[3];
        volatile double u = 1.0 - rr;
        volatile double su = std::sqrt((double)u);
        volatile double sq = std::sqrt(c->dt);
        a.sc.rc = su * sq;
        a.sqdt = sq;
        // tangent mode: d rho_comp / d rho = -rho * sqrt(dt) / sqrt(1 - rho^2)
        // (0 where the sqrt's argument is 0: the tape's sqrt-at-0 convention)
        a.drc = su > 0.0 ? -(x[3] * sq) / su : 0.0;
    }
    a.sc.dt = c->dt;
    a.sc.sqdt = a.sqdt;
    a.sc.mu_dt = a.mu_dt;
    a.sc.half_dt = a.half_dt;
    a.scf = to_float(a.sc);
    a.x = c->x_src;
    a.v0 = x[4];
    if (c->nlev <= (uint32_t)kInlineLev) {
        a.lev_inline = 1;
        std::copy(x + 5, x + 5 + c->nlev, a.lev_in);
    }
    a.s_nodes = c->d_snodes.as<double>();
    a.row_off = c->d_rowoff.as<uint16_t>();
    a.events = c->d_events.as<MaturityEvent>();
    a.inst_order = c->d_order.as<uint32_t>();
    a.strike = c->d_strike.as<double>();
    a.kind = c->d_kind.as<int32_t>();
    a.tables = c->d_tab.as<RngTables>();
    a.rc = c->h_rc;
    a.seg_steps = c->seg_steps;
    // plain Heston (one leverage cell equal to 1.0): the kLevUnit kernels skip
    // the exact products by L (LTG_UNIT_LEV=0: the general kernels, tests)
    static const bool unit_ok = [] {
        const char* e = std::getenv("LTG_UNIT_LEV");
        return !(e && e[0] == '0');
    }();
    a.unit_lev = (unit_ok && c->nlev == 1 && x[5] == 1.0) ? 1 : 0;
    a.fp32 = c->fp32;
    a.safe = c->safe;
    a.rare = rare_ptr(c);
    a.rare_thr = kRareThr;
    if (c->draws_on) {
        a.draws = c->d_draws.as<double>();
        a.draws_row0 = c->draws_row0A;
    }
    return a;
}

// Pass 2's input table for `stride` paths (heston.cu): grid layouts keep
// (S, V) at every checkpoint; one-column layouts (the S-free pass 2) keep V
// at every checkpoint and S at every maturity event.
struct TabLayout {
    size_t ck_bytes, smat_off, total;
};
bool s_free(const ltg_ctx* c) { return c->kind == 0 && c->cols == 1; }
TabLayout tab_layout(const ltg_ctx* c, uint32_t ks, uint64_t stride) {
    const size_t r = c->fp32 ? 4 : 8;
    const uint32_t nseg = (c->steps + ks - 1) / ks;
    const size_t rows = nseg > 1 ? nseg - 1 : 0;
    TabLayout t{};
    if (!s_free(c)) {
        t.ck_bytes = rows * stride * 2 * r;
        t.smat_off = t.total = t.ck_bytes;
    } else {
        t.ck_bytes = rows * stride * r;
        t.smat_off = (t.ck_bytes + 255) & ~size_t(255);
        t.total = t.smat_off + c->events.size() * stride * r;
    }
    return t;
}

// Test knob LTG_TEST_FRESH_RARE=1: the range check of the fresh step-2 path
// set (and only it) flags every path, which forces the exact rerun that a
// genuinely out-of-range fresh-path argument would (tests/test_gpu_parity.py)
unsigned fresh_check_thr() {
    const char* e = std::getenv("LTG_TEST_FRESH_RARE");
    return (e && e[0] == '1') ? 0u : kRareThr;
}

Work base_work(ltg_ctx* c, const ltg_mc_config& cfg, const ltg_shard& plan) {
    Work w{};
    w.paths = cfg.paths;
    w.path_offset = c->path_base;
    w.chunk_paths = plan.chunk_paths;
    w.chunk_begin = plan.chunk_begin;
    w.n_chunks = plan.chunk_end - plan.chunk_begin;
    w.ckpt_path0 = plan.path_begin;
    w.ckpt_stride = std::max<uint64_t>(1, plan.path_end - plan.path_begin);
    w.counter = counter_ptr(c, 0);
    w.rk = make_philox_keys((uint32_t)cfg.seed, (uint32_t)(cfg.seed >> 32));
    // (caller draws: no antithetic pairing, so the kernels' Philox path word
    // is the path index, which also addresses the caller's row)
    w.antithetic = cfg.antithetic && !c->draws_on ? 1 : 0;
    return w;
}

// Enqueue helpers of a call's non-kernel device work (see GraphRec).
void enq_memset(ltg_ctx* c, void* p, size_t n) {
    if (t_rec && !t_rec->op(0, p, nullptr, n)) return;
    cuda_check(cudaMemsetAsync(p, 0, n, c->stream), "memset");
}
void enq_copy(ltg_ctx* c, void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
    if (t_rec && !t_rec->op(1 + (int)kind, dst, src, n)) return;
    cuda_check(cudaMemcpyAsync(dst, src, n, kind, c->stream), "copy");
}
void rec_event(ltg_ctx* c, int i) {
    c->ev_at[i] = i;
    if (!c->timing_on) return;  // (ltg_set_timing: no events; the device times read 0)
    if (t_rec && !t_rec->op(16, c->ev[i], nullptr, 0)) return;
    // (inside a capture: an event-record node, so the timing events work on replay)
    cuda_check(t_rec ? cudaEventRecordWithFlags(c->ev[i], c->stream, cudaEventRecordExternal)
                     : cudaEventRecord(c->ev[i], c->stream),
               "event");
}
// timing point i is where point j was recorded (nothing enqueued between)
void same_event(ltg_ctx* c, int i, int j) { c->ev_at[i] = c->ev_at[j]; }

void validate_cfg(ltg_ctx* c, const ltg_mc_config* cfg, size_t M) {
    require(cfg != nullptr, "null MCConfig");
    require_f(M == c->M, [&] {
        return "parameter vector has " + std::to_string(M) + " entries, program has " +
               std::to_string(c->M);
    });
    require(cfg->paths > 0, "forward_pass: paths must be > 0");
    require(cfg->precision == LTG_FP64 || cfg->precision == LTG_FP32, "unknown precision");
    require(cfg->precision == LTG_FP64 || c->kind == 0,
            "fp32 precision is implemented for Heston-SLV programs (config 5)");
    c->fp32 = cfg->precision == LTG_FP32 ? 1 : 0;
}

// The one EvalError site of the recorded Heston program: rho_comp's sqrt of
// 1 - rho^2 (heston.hpp:286) throws for a negative argument (tape.hpp:261-263,
// kernel.hpp "sqrt of negative value"; NaN passes the a < 0 test). Nothing
// else in either model can throw: non-finite parameters or results propagate
// into the report as in the reference library, whose gradient_of_G /
// estimate_means return them (only its CLI refuses them, main.cpp
// require_finite).
void check_params(ltg_ctx* c, const double* x) {
    if (c->kind == 0 && 1.0 - x[3] * x[3] < 0.0)
        throw Failure(LTG_ENUMERIC, "sqrt of negative value (1 - rho^2)");
}

// Pass 1 over this rank's chunks (+ all-gather) and the fixed-order reduction
// into d_res = [G, means, se, lambda]. Returns whether pass-2 checkpoints of the
// step-1 path set were written.
bool run_pass1(ltg_ctx* c, const ltg_mc_config& cfg, const ltg_shard& plan, bool targets,
               bool want_ckpt, bool last = false) {
    const uint64_t per = chunks_per_rank(plan, c->world);
    const uint64_t table_rows = per * c->world;
    const uint32_t width = 2 * c->m;
    c->d_part1.ensure(table_rows * width * 8);
    c->d_groups.ensure(((plan.n_chunks + kGroup - 1) / kGroup) * std::max(width, c->M) * 8 + 8);
    c->d_tot1.ensure(width * 8);

    Work w = base_work(c, cfg, plan);
    Finish fin{};
    fin.means = 1;
    fin.m = c->m;
    fin.paths = cfg.paths;
    if (targets) set_targets(c, fin);
    fin.res = res_ptr(c);
    if (last) set_pub(c, fin);  // (estimate_means: pass 1 ends the call)
    const bool fused = fuse_reduce(c, w, width, c->d_tot1.as<double>(), fin);
    if (c->kind == 1) {
        // basket: (S, W) at every maturity for pass 2 (store mode) when it fits
        BasketArgs b = basket_args(c, c->h_x.data());
        c->store_ok = false;
        if (want_ckpt) {
            const size_t need = size_t(b.n_events) * b.n * w.ckpt_stride * 16;
            size_t free_b = 0, total_b = 0;
            if (need > c->d_ckpt.bytes) cudaMemGetInfo(&free_b, &total_b);
            if (need <= c->d_ckpt.bytes || need + (size_t(2) << 30) < free_b) {
                c->d_ckpt.ensure(need);
                c->store_ok = true;
            }
        }
        b.partials = c->d_part1.as<double>() + plan.chunk_begin * width;
        b.store = c->store_ok ? c->d_ckpt.as<double2>() : nullptr;
        b.store_stride = w.ckpt_stride;
        b.write_sums = 1;
        b.write_store = c->store_ok ? 1 : 0;
        rec_event(c, 0);
        if (w.n_chunks) cuda_check(launch_basket_pass1(b, w, 0, c->stream), "basket pass 1");
        rec_event(c, 1);
        c->timing.launches += w.n_chunks ? 1 : 0;
    }
    // HBM plan for pass 2's inputs: the state every KS steps,
    // plus the draws of as many chunks as fit (pass 2 then reads them instead
    // of regenerating them): KS = 8 if its table fits, else KS = 16, else no
    // table (pass 2 replays its checkpoints in waves). LTG_CKPT_STEPS /
    // LTG_ZSTORE=0 override (tuning).
    bool ckpt = false;
    c->seg_steps = 16;
    c->z_chunks = 0;
    auto env_or = [](const char* k) {
        const char* v = std::getenv(k);
        return std::string(v ? v : "-");
    };
    const std::string key =
        want_ckpt && c->kind == 0
            ? std::to_string(cfg.paths) + "/" + std::to_string(w.n_chunks) + "/" +
                  std::to_string(plan.chunk_paths) + "/" + std::to_string(w.ckpt_stride) + "/" +
                  std::to_string(c->fp32) + "/" + std::to_string(c->hbm_budget) + "/" +
                  env_or("LTG_HBM_BUDGET_GB") + "/" + env_or("LTG_CKPT_STEPS") + "/" +
                  env_or("LTG_ZSTORE") + "/" + env_or("LTG_ZCHUNKS_MAX") + "/" +
                  std::to_string(c->draws_on ? 1 : 0)
            : std::string();
    if (!key.empty() && key == c->plan_key) {
        c->seg_steps = c->plan_ks;
        c->z_chunks = c->plan_z;
        ckpt = c->plan_chosen && (s_free(c) || ((c->steps + c->seg_steps - 1) / c->seg_steps) > 1);
        if (!ckpt) c->z_chunks = 0;
    } else if (want_ckpt && c->kind == 0) {
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        const size_t reserve = size_t(2) << 30;
        const size_t held = c->d_ckpt.bytes + c->d_ztab.bytes;
        size_t avail = free_b + held > reserve ? free_b + held - reserve : 0;
        // LTG_HBM_BUDGET_GB caps checkpoint table + draw store (GPUs shared
        // with other work); the default takes what is free
        if (const char* cap = std::getenv("LTG_HBM_BUDGET_GB"))
            avail = std::min<size_t>(avail, size_t(std::strtod(cap, nullptr) * double(1ull << 30)));
        if (c->hbm_budget) avail = std::min<size_t>(avail, c->hbm_budget);
        const size_t elem = c->fp32 ? 8 : 16;
        const uint64_t nloc = w.n_chunks;
        const size_t z_chunk = size_t(c->steps) * plan.chunk_paths * elem;
        auto ck_bytes = [&](uint32_t ks) { return tab_layout(c, ks, w.ckpt_stride).total; };
        const char* env_ks = std::getenv("LTG_CKPT_STEPS");
        const char* env_z = std::getenv("LTG_ZSTORE");
        // (caller draws: pass 2 reads the caller's rows, nothing to store)
        const bool z_ok = !(env_z && env_z[0] == '0') && !c->draws_on;
        const uint32_t forced = env_ks ? (uint32_t)std::atoi(env_ks) : 0u;
        // the first interval whose checkpoint table fits, with the draws of as
        // many chunks as the rest of HBM holds (KS = 8 halves the replay
        // buffers of KS = 16 and keeps 5 pass-2 CTAs per SM resident)
        bool chosen = false;
        for (uint32_t ks : {8u, 16u}) {
            if (forced && ks != forced) continue;
            if (ck_bytes(ks) > avail) continue;
            c->seg_steps = ks;
            c->z_chunks = z_ok ? std::min<uint64_t>(nloc, (avail - ck_bytes(ks)) / z_chunk) : 0;
            chosen = true;
            break;
        }
        if (const char* cap = std::getenv("LTG_ZCHUNKS_MAX"))  // tests: partial draw store
            c->z_chunks = std::min<uint64_t>(c->z_chunks, std::strtoull(cap, nullptr, 10));
        if (chosen) {
            const size_t need_ck = ck_bytes(c->seg_steps);
            const size_t need_z = size_t(c->z_chunks) * z_chunk;
            if (need_ck > c->d_ckpt.bytes || need_z > c->d_ztab.bytes) {
                c->d_ckpt.release();
                c->d_ztab.release();
                c->d_ckpt.ensure(need_ck);
                c->d_ztab.ensure(need_z);
            }
            ckpt = s_free(c) || ((c->steps + c->seg_steps - 1) / c->seg_steps) > 1;
            if (!ckpt) c->z_chunks = 0;
        }
        c->plan_key = key;
        c->plan_ks = c->seg_steps;
        c->plan_z = c->z_chunks;
        c->plan_chosen = chosen;
    }
    if (c->kind == 0) {
        HestonArgs a = heston_args(c, c->h_x.data());
        // partial rows are indexed from the launch's first chunk
        a.partials = c->d_part1.as<double>() + plan.chunk_begin * width;
        a.ckpt = ckpt ? c->d_ckpt.p : nullptr;
        a.smat = ckpt ? c->d_ckpt.as<char>() + tab_layout(c, c->seg_steps, w.ckpt_stride).smat_off
                      : nullptr;
        a.write_sums = 1;
        a.write_ckpt = ckpt ? 1 : 0;
        a.ztab = c->d_ztab.p;
        a.z_chunks = c->z_chunks;
        a.z_stride = std::max<uint64_t>(1, c->z_chunks * plan.chunk_paths);
        a.write_z = c->z_chunks > 0 ? 1 : 0;
        rec_event(c, 0);
        if (w.n_chunks) cuda_check(launch_heston_pass1(a, w, 0, c->stream), "heston pass 1");
        rec_event(c, 1);
        c->timing.launches += w.n_chunks ? 1 : 0;
    } else {
        ckpt = c->store_ok;
    }
    if (!fused) {
        all_gather_rows(c, c->d_part1.as<double>(), per, width);
        cuda_check(launch_reduce_chunks(c->d_part1.as<double>(), plan.n_chunks, width,
                                        c->d_groups.as<double>(), c->d_tot1.as<double>(), fin,
                                        c->stream),
                   "reduce");
        c->timing.launches += reduce_launch_count(plan.n_chunks);
        rec_event(c, 2);
    } else {
        same_event(c, 2, 1);
    }
    c->timing.paths_pass1 = plan.path_end - plan.path_begin;
    if (ckpt && c->kind == 0) {
        c->timing.seg_steps = c->seg_steps;
        c->timing.ckpt_bytes = tab_layout(c, c->seg_steps, w.ckpt_stride).total;
        c->timing.z_bytes = c->z_chunks * plan.chunk_paths * c->steps * (c->fp32 ? 8 : 16);
    } else if (ckpt) {
        c->timing.ckpt_bytes = uint64_t(c->events.size()) * c->n_assets * w.ckpt_stride * 16;
    }
    return ckpt;
}

// chained: enqueued right behind run_pass1 (its last timing point is pass 2's start)
void run_pass2(ltg_ctx* c, const ltg_mc_config& cfg, const ltg_shard& plan, bool have_ckpt,
               bool chained = false) {
    const uint64_t per = chunks_per_rank(plan, c->world);
    const uint64_t table_rows = per * c->world;
    c->d_part2.ensure(table_rows * c->M * 8);
    c->d_tot2.ensure(c->M * 8);
    // caller draws: pass 2 reads the rows of its own path set (the fresh
    // step-2 rows follow the pass-1 rows in d_draws)
    const bool fresh_rows = c->draws_on && cfg.fresh_step2_paths;
    const double* p2_draws =
        c->draws_on ? c->d_draws.as<double>() + (fresh_rows ? c->draws_rowsA * c->N : 0)
                    : nullptr;
    const uint64_t p2_row0 = fresh_rows ? c->draws_row0B : c->draws_row0A;
    // (the Heston argument block reads x[0..5]: built for Heston contexts only)
    HestonArgs a = c->kind == 0 ? heston_args(c, c->h_x.data()) : HestonArgs{};
    a.lambda = res_ptr(c) + 1 + 2 * c->m;
    a.draws = p2_draws;
    a.draws_row0 = p2_row0;
    Work w = base_work(c, cfg, plan);
    Finish fin{};
    fin.grad = 1;
    fin.M = (uint32_t)c->M;
    fin.paths = cfg.paths;
    fin.grad_out = grad_ptr(c);
    set_pub(c, fin);
    bool fused = false;
    const uint32_t nseg = (c->steps + c->seg_steps - 1) / c->seg_steps;
    if (chained)
        same_event(c, 3, 2);
    else
        rec_event(c, 3);
    if (w.n_chunks && c->kind == 1) {
        BasketArgs b = basket_args(c, c->h_x.data());
        b.lambda = res_ptr(c) + 1 + 2 * c->m;
        b.draws = p2_draws;
        b.draws_row0 = p2_row0;
        b.partials = c->d_part2.as<double>() + plan.chunk_begin * c->M;
        b.use_store = have_ckpt && !cfg.fresh_step2_paths ? 1 : 0;
        b.store = b.use_store ? c->d_ckpt.as<double2>() : nullptr;
        b.store_stride = w.ckpt_stride;
        if (cfg.fresh_step2_paths) w.path_offset += cfg.paths;
        w.counter = counter_ptr(c, 2);
        fused = fuse_reduce(c, w, c->M, c->d_tot2.as<double>(), fin);
        cuda_check(launch_basket_pass2(b, w, 0, c->stream), "basket pass 2");
        c->timing.launches += 1;
    } else if (w.n_chunks) {
        const bool sf = s_free(c);
        if (!have_ckpt && (nseg > 1 || sf)) {
            // fresh_step2_paths or no room for a full checkpoint table: replay
            // the pass-2 path set in waves (checkpoint-only forward, then adjoint)
            if (cfg.fresh_step2_paths) w.path_offset += cfg.paths;
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            const size_t per_chunk = tab_layout(c, c->seg_steps, plan.chunk_paths).total + 256;
            size_t budget = c->d_ckpt.bytes;
            if (budget < per_chunk * 64 && free_b > (size_t(2) << 30))
                budget = std::max(budget, std::min(free_b - (size_t(2) << 30),
                                                   per_chunk * w.n_chunks));
            if (c->hbm_budget) budget = std::min<size_t>(budget, c->hbm_budget);  // >= 1 chunk below
            uint64_t wave = std::max<uint64_t>(1, budget / per_chunk);
            wave = std::min<uint64_t>(wave, w.n_chunks);
            c->d_ckpt.ensure(wave * per_chunk);
            for (uint64_t c0 = 0; c0 < w.n_chunks; c0 += wave) {
                Work ww = w;
                ww.chunk_begin = w.chunk_begin + c0;
                ww.n_chunks = std::min<uint64_t>(wave, w.n_chunks - c0);
                ww.ckpt_path0 = ww.chunk_begin * plan.chunk_paths;
                ww.ckpt_stride = ww.n_chunks * plan.chunk_paths;
                const size_t smat_off = tab_layout(c, c->seg_steps, ww.ckpt_stride).smat_off;
                HestonArgs r = a;
                r.ckpt = c->d_ckpt.p;
                r.smat = c->d_ckpt.as<char>() + smat_off;
                r.write_sums = 0;
                r.write_ckpt = 1;
                r.partials = nullptr;
                // every step: the S-free layout needs S at every maturity, and
                // no forward has range-checked the fresh path set
                r.check_all = (sf || cfg.fresh_step2_paths) ? 1 : 0;
                if (cfg.fresh_step2_paths) r.rare_thr = fresh_check_thr();
                ww.counter = counter_ptr(c, 1);
                cuda_check(launch_heston_pass1(r, ww, 0, c->stream), "heston replay");
                HestonArgs b = a;
                b.ckpt = c->d_ckpt.p;
                b.smat = c->d_ckpt.as<char>() + smat_off;
                b.partials = c->d_part2.as<double>() + ww.chunk_begin * c->M;
                ww.counter = counter_ptr(c, 2);
                cuda_check(launch_heston_pass2(b, ww, 0, c->stream), "heston pass 2");
                c->timing.launches += 2;
            }
        } else {
            if (cfg.fresh_step2_paths) {
                w.path_offset += cfg.paths;
                if (!c->safe) {  // (safe kernels compute no flag)
                    // one segment (steps <= KS): no checkpoint replay ran over
                    // the fresh paths, so range-check them with a forward first
                    HestonArgs r = a;
                    r.write_sums = 0;
                    r.write_ckpt = 0;
                    r.ckpt = nullptr;
                    r.partials = nullptr;
                    r.check_all = 1;
                    r.rare_thr = fresh_check_thr();
                    Work ww = w;
                    ww.counter = counter_ptr(c, 1);
                    cuda_check(launch_heston_pass1(r, ww, 0, c->stream), "heston range check");
                    c->timing.launches += 1;
                }
            }
            a.ckpt = c->d_ckpt.p;
            a.smat = c->d_ckpt.as<char>() + tab_layout(c, c->seg_steps, w.ckpt_stride).smat_off;
            a.ztab = c->d_ztab.p;
            a.z_chunks = c->z_chunks;
            a.z_stride = std::max<uint64_t>(1, c->z_chunks * plan.chunk_paths);
            a.use_z = (c->z_chunks > 0 && !cfg.fresh_step2_paths) ? 1 : 0;
            a.partials = c->d_part2.as<double>() + plan.chunk_begin * c->M;
            w.counter = counter_ptr(c, 2);
            fused = fuse_reduce(c, w, c->M, c->d_tot2.as<double>(), fin);
            cuda_check(launch_heston_pass2(a, w, 0, c->stream), "heston pass 2");
            c->timing.launches += 1;
        }
    }
    rec_event(c, 4);
    if (!fused) {
        all_gather_rows(c, c->d_part2.as<double>(), per, c->M);
        cuda_check(launch_reduce_chunks(c->d_part2.as<double>(), plan.n_chunks, c->M,
                                        c->d_groups.as<double>(), c->d_tot2.as<double>(), fin,
                                        c->stream),
                   "reduce");
        c->timing.launches += reduce_launch_count(plan.n_chunks);
        rec_event(c, 5);
    } else {
        same_event(c, 5, 4);
    }
    c->timing.paths_pass2 = plan.path_end - plan.path_begin;
}

// Tangent mode (ltg_gradient_of_G_tangent): one forward launch over the
// pass-2 path set carrying the parameter tangents; rows [sum | sumsq | J].
// With `sums` the same launch also provides pass 1 (means, lambda, G);
// otherwise (fresh_step2_paths) pass 1 ran before and only J is used.
void run_tangent(ltg_ctx* c, const ltg_mc_config& cfg, const ltg_shard& plan, bool sums) {
    const uint64_t per = chunks_per_rank(plan, c->world);
    const uint64_t table_rows = per * c->world;
    const uint32_t width = 2 * c->m + c->m * (uint32_t)c->M;
    c->d_part2.ensure(table_rows * width * 8);
    c->d_groups.ensure(((plan.n_chunks + kGroup - 1) / kGroup) * width * 8 + 8);
    c->d_tot2.ensure(width * 8);
    HestonArgs a = heston_args(c, c->h_x.data());
    a.partials = c->d_part2.as<double>() + plan.chunk_begin * width;
    a.write_sums = sums ? 1 : 0;
    Work w = base_work(c, cfg, plan);
    if (cfg.fresh_step2_paths) w.path_offset += cfg.paths;
    w.counter = counter_ptr(c, 2);
    // one finishing step: (means, lambda, G when this launch is pass 1) then
    // grad = sum_i lambda_i J_i / P
    Finish fin{};
    fin.means = sums ? 1 : 0;
    fin.grad_tangent = 1;
    fin.m = c->m;
    fin.M = (uint32_t)c->M;
    fin.paths = cfg.paths;
    set_targets(c, fin);
    fin.res = res_ptr(c);
    fin.grad_out = grad_ptr(c);
    set_pub(c, fin);
    const bool fused = fuse_reduce(c, w, width, c->d_tot2.as<double>(), fin);
    rec_event(c, sums ? 0 : 3);
    if (w.n_chunks) cuda_check(launch_heston_tangent(a, w, 0, c->stream), "heston tangent");
    rec_event(c, sums ? 1 : 4);
    c->timing.launches += w.n_chunks ? 1 : 0;
    if (!fused) {
        all_gather_rows(c, c->d_part2.as<double>(), per, width);
        cuda_check(launch_reduce_chunks(c->d_part2.as<double>(), plan.n_chunks, width,
                                        c->d_groups.as<double>(), c->d_tot2.as<double>(), fin,
                                        c->stream),
                   "reduce");
        c->timing.launches += reduce_launch_count(plan.n_chunks);
        rec_event(c, 5);
    } else {
        same_event(c, 5, sums ? 1 : 4);
    }
    if (sums) {  // (pass 1 and the gradient in one launch: no pass-2 span)
        c->timing.paths_pass1 = plan.path_end - plan.path_begin;
        same_event(c, 2, 5);
        same_event(c, 3, 5);
        same_event(c, 4, 5);
    }
    c->timing.paths_pass2 = plan.path_end - plan.path_begin;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// The device times of the last call, read from its events when asked for
// (ltg_last_timing) rather than inside the call: seven event queries cost
// more than the whole host side of a replayed small call.
void settle_timing(ltg_ctx* c) {
    auto E = [c](int i) { return c->ev[c->ev_at[i]]; };
    if (!c->timing_on) c->timing_pending = 0;
    if (c->timing_pending == 1) {  // gradient_of_G: pass 1, pass 2, both reductions
        c->timing.pass1_ms = elapsed(E(0), E(1));
        c->timing.pass2_ms = elapsed(E(3), E(4));
        c->timing.reduce_ms = elapsed(E(1), E(2)) + elapsed(E(4), E(5));
        c->timing.total_ms = elapsed(E(0), E(5));
    } else if (c->timing_pending == 2) {  // estimate_means: pass 1 and its reduction
        c->timing.pass1_ms = elapsed(E(0), E(1));
        c->timing.reduce_ms = elapsed(E(1), E(2));
        c->timing.total_ms = elapsed(E(0), E(2));
    }
    c->timing_pending = 0;
}

// The fast arithmetic's out-of-range flag (heston.cu heston_step): cleared
// before a call, OR-ed across ranks, copied back with the results. A set flag
// makes the caller redo the call in safe mode.
// Calls start in fast mode unless LTG_SAFE=1 (tests) or the host libm's exp
// table could not be validated: the fast kernels use glibc's exp main path
// unconditionally, so without an exact table every call runs the SAFE
// kernels (which fall back to CUDA's exp).
int start_safe(const ltg_ctx* c) {
    const char* e = std::getenv("LTG_SAFE");
    return (e && e[0] == '1') || !c->h_rc.exact_exp ? 1 : 0;
}

// One memset at the start of a call: the rare flag (and the scheduler slots,
// which their launches leave zero anyway). The call's kernels may set the
// flag again; only a lean call's last kernel clears it (flag_clean).
void reset_flags(ltg_ctx* c) {
    enq_memset(c, flags_ptr(c), kFlagWords * 4);
    c->flag_clean = false;
}

// The rare flag after the call's kernels: all-reduced over the ranks (NCCL);
// it reaches the host with the report (copy_out), or alone (copy_rare), and
// is read once the stream is done (wait_rare; loopback members exchange it
// on the host instead).
void reduce_rare(ltg_ctx* c) {
    uint32_t* d = rare_ptr(c);
    if (c->comm && !c->loop) {
        const ncclResult_t r = nccl().AllReduce(d, d, 1, ncclUint32, ncclMax, c->comm, c->stream);
        if (r != ncclSuccess)
            throw Failure(LTG_ECUDA, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
    }
}
// the report [G, means, se, lambda, grad] and the rare flag in one copy; the
// flag lands at host + out_doubles(c)
void copy_out(ltg_ctx* c, double* host) {
    reduce_rare(c);
    enq_copy(c, host, res_ptr(c), out_doubles(c) * 8 + 4, cudaMemcpyDeviceToHost);
}
void copy_rare(ltg_ctx* c, double* host_slot) {
    reduce_rare(c);
    enq_copy(c, host_slot, rare_ptr(c), 4, cudaMemcpyDeviceToHost);
}

bool wait_rare(ltg_ctx* c, const double* host_slot) {
    cuda_check(cudaStreamSynchronize(c->stream), "synchronize");
    uint32_t v = 0;
    std::memcpy(&v, host_slot, sizeof v);
    if (c->loop) {
        Loopback& L = *c->loop;
        L.flags[c->rank] = v;
        L.barrier();
        for (uint32_t f : L.flags) v = std::max(v, f);
        L.barrier();
    }
    return v != 0;
}

// The call's x and targets. The kernels take v0, the leverage cells and the
// targets by value when they fit (HestonArgs::lev_in, Finish::tgt_in); only
// larger models copy [x | targets] to d_x (one H2D copy from the pinned
// staging area).
void upload_x(ltg_ctx* c, const double* x, const double* targets) {
    c->h_x.assign(x, x + c->M);
    if (targets)
        c->h_t.assign(targets, targets + c->m);
    else
        c->h_t.clear();
    const bool fits = (c->kind != 0 || c->nlev <= (uint32_t)kInlineLev) &&
                      (!targets || c->m <= (uint32_t)kInlineTargets);
    if (fits) {
        c->x_src = nullptr;
        return;
    }
    const size_t n = c->M + (targets ? c->m : 0);
    double* st = c->stage(n);
    std::memcpy(st, x, c->M * 8);
    if (targets) std::memcpy(st + c->M, targets, c->m * 8);
    c->d_x.ensure((c->M + c->m) * 8);  // [x | targets]: one copy
    enq_copy(c, c->d_x.p, st, n * 8, cudaMemcpyHostToDevice);
    c->x_src = c->d_x.as<double>();
}

// the targets of a finishing launch: by value, or behind x in d_x
void set_targets(ltg_ctx* c, Finish& fin) {
    if (c->h_t.empty()) return;
    if (c->m <= (uint32_t)kInlineTargets) {
        fin.tgt_inline = 1;
        std::copy(c->h_t.begin(), c->h_t.end(), fin.tgt_in);
    } else {
        fin.targets = c->x_src + c->M;
    }
}

// the report of a lean call (its last reduction publishes it, Finish::pub)
void set_pub(ltg_ctx* c, Finish& fin) {
    if (!c->pub) return;
    fin.pub = c->pub;
    fin.pub_src = res_ptr(c);
    fin.pub_n = (uint32_t)out_doubles(c);
    fin.rare = rare_ptr(c);
}

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("LTG_GRAPH");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Runs the enqueue sequence `body` of one call: eagerly; or, for a
// single-GPU context whose call of shape `key` arrives the second time in a
// row, captured into a graph and launched; or, for later calls of that
// shape, as an update of the graph followed by one cudaGraphLaunch (GraphRec).
void run_body(ltg_ctx* c, bool graphable, const std::string& key,
              const std::function<void()>& body) {
    if (!graphable || !graphs_enabled()) {
        body();
        return;
    }
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {  // first call of this shape: eager (allocates, plans)
        constexpr size_t kMaxGraphs = 8;
        if (c->graph_order.size() == kMaxGraphs) {
            c->graphs.erase(c->graph_order.front());
            c->graph_order.erase(c->graph_order.begin());
        }
        c->graphs.emplace(key, std::make_unique<GraphRec>());
        c->graph_order.push_back(key);
        body();
        return;
    }
    GraphRec& g = *it->second;
    struct Hook {
        explicit Hook(GraphRec* r) { t_rec = r; t_launch_hook = r; }
        ~Hook() { t_rec = nullptr; t_launch_hook = nullptr; }
    };
    if (g.exec && g.key == key) {
        const ltg_timing saved = c->timing;
        g.mode = GraphRec::Update;
        g.kcur = g.ocur = 0;
        g.mismatch = false;
        {
            Hook h(&g);
            body();
        }
        if (!g.mismatch && g.kcur == g.kernels.size() && g.ocur == g.ops.size()) {
            cuda_check(cudaGraphLaunch(g.exec, c->stream), "cudaGraphLaunch");
            c->timing.graph = 2;
            return;
        }
        g.reset();  // the call's shape changed under the same key: eager, recapture next time
        c->timing = saved;
        body();
        return;
    }
    g.reset();
    g.mode = GraphRec::Capture;
    cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "capture");
    try {
        Hook h(&g);
        body();
    } catch (...) {
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(c->stream, &dead);
        if (dead) cudaGraphDestroy(dead);
        cudaGetLastError();
        g.reset();
        throw;
    }
    cuda_check(cudaStreamEndCapture(c->stream, &g.graph), "end capture");
    // the capture of one stream is a chain: its kernel nodes in launch order
    size_t nroot = 0;
    cuda_check(cudaGraphGetRootNodes(g.graph, nullptr, &nroot), "graph roots");
    std::vector<cudaGraphNode_t> cur(nroot);
    cuda_check(cudaGraphGetRootNodes(g.graph, cur.data(), &nroot), "graph roots");
    while (cur.size() == 1) {
        cudaGraphNodeType t;
        cuda_check(cudaGraphNodeGetType(cur[0], &t), "node type");
        if (t == cudaGraphNodeTypeKernel) g.knodes.push_back(cur[0]);
        size_t nd = 0;
        cuda_check(cudaGraphNodeGetDependentNodes(cur[0], nullptr, &nd), "dependents");
        std::vector<cudaGraphNode_t> next(nd);
        if (nd) cuda_check(cudaGraphNodeGetDependentNodes(cur[0], next.data(), &nd), "dependents");
        cur.swap(next);
    }
    if (!cur.empty() || g.knodes.size() != g.kernels.size()) {
        // not the expected chain: run this call from the captured graph
        // once, keep no graph
        cudaGraphExec_t once = nullptr;
        cuda_check(cudaGraphInstantiate(&once, g.graph, 0), "instantiate");
        cuda_check(cudaGraphLaunch(once, c->stream), "cudaGraphLaunch");
        cuda_check(cudaStreamSynchronize(c->stream), "synchronize");
        cudaGraphExecDestroy(once);
        g.reset();
        return;
    }
    cuda_check(cudaGraphInstantiate(&g.exec, g.graph, 0), "instantiate");
    g.key = key;
    cuda_check(cudaGraphLaunch(g.exec, c->stream), "cudaGraphLaunch");
    c->timing.graph = 1;
}

}  // namespace

namespace {

// ltg_create_*_devices: one member context per device plus ncclCommInitAll
template <typename Create>
int create_group(const int* devices, int n, ltg_ctx** out, Create create) {
    if (!out || !devices || n < 1) {
        g_create_error = "create_devices: need an output pointer and >= 1 device";
        return LTG_EINVAL;
    }
    *out = nullptr;
    const char* lb = std::getenv("LTG_LOOPBACK");
    const bool loopback = lb && lb[0] == '1';  // tests: members may share a device
    auto g = std::make_unique<ltg_ctx>();
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < i && !loopback; ++j)
            if (devices[j] == devices[i]) {
                g_create_error = "create_devices: a device may appear once";
                return LTG_EINVAL;
            }
        ltg_ctx* m = nullptr;
        const int rc = create(devices[i], &m);
        if (rc != LTG_OK) return rc;  // g_create_error set by the member's create
        g->members.emplace_back(m);
    }
    if (loopback) {
        auto L = std::make_shared<Loopback>(n);
        for (int i = 0; i < n; ++i) {
            g->members[i]->loop = L;
            g->members[i]->rank = i;
            g->members[i]->world = n;
        }
    } else {
    std::string why;
    if (!nccl().load(why)) {
        g_create_error = why;
        return LTG_ECUDA;
    }
    std::vector<ncclComm_t> comms(n);
    const ncclResult_t r = nccl().CommInitAll(comms.data(), n, devices);
    if (r != ncclSuccess) {
        g_create_error = std::string("ncclCommInitAll: ") + nccl().GetErrorString(r);
        return LTG_ECUDA;
    }
    for (int i = 0; i < n; ++i) {
        g->members[i]->comm = comms[i];
        g->members[i]->rank = i;
        g->members[i]->world = n;
    }
    }
    const ltg_ctx& m0 = *g->members[0];
    g->kind = m0.kind;
    g->M = m0.M;
    g->m = m0.m;
    g->N = m0.N;
    g->x0 = m0.x0;
    g->h_rc = m0.h_rc;
    g->device = m0.device;
    *out = g.release();
    return LTG_OK;
}

}  // namespace

extern "C" {

int ltg_abi_version(void) { return LTG_ABI_VERSION; }

int ltg_create_heston(const ltg_heston_model* mdl, int device, ltg_ctx** out) {
    if (!out || !mdl) {
        g_create_error = "null argument";
        return LTG_EINVAL;
    }
    *out = nullptr;
    auto c = std::make_unique<ltg_ctx>();
    const int rc = guarded(c.get(), [&] {
        const ltg_heston_model& m = *mdl;
        // validate(ModelSpec) minus McSettings.paths (heston.hpp:30-130)
        require(m.s0 > 0.0, "HestonParams: s0 must be > 0");
        require(m.v0 >= 0.0, "HestonParams: v0 must be >= 0");
        require(m.theta >= 0.0, "HestonParams: theta must be >= 0");
        require(m.kappa >= 0.0, "HestonParams: kappa must be >= 0");
        require(m.xi >= 0.0, "HestonParams: xi must be >= 0");
        require(std::fabs(m.rho) < 1.0, "HestonParams: rho must satisfy |rho| < 1");
        require(std::isfinite(m.mu), "HestonParams: mu must be finite");
        require(m.n_t_nodes > 0 && m.n_s_nodes > 0 && m.t_nodes && m.s_nodes,
                "LeverageGrid: node lists must be non-empty");
        for (uint32_t i = 1; i < m.n_t_nodes; ++i)
            require(m.t_nodes[i] > m.t_nodes[i - 1], "LeverageGrid: t_nodes must be strictly ascending");
        for (uint32_t i = 1; i < m.n_s_nodes; ++i)
            require(m.s_nodes[i] > m.s_nodes[i - 1], "LeverageGrid: s_nodes must be strictly ascending");
        const uint32_t nlev = m.n_t_nodes * m.n_s_nodes;
        require(m.leverage != nullptr, "LeverageGrid: values must hold t_nodes x s_nodes entries");
        for (uint32_t i = 0; i < nlev; ++i)
            require(std::isfinite(m.leverage[i]) && m.leverage[i] >= 0.0,
                    "LeverageGrid: values must be finite and >= 0");
        require(m.steps > 0, "mc: steps must be > 0");
        require(m.dt > 0.0, "mc: dt must be > 0");
        require(m.n_instruments > 0, "instruments: list must be non-empty");
        for (uint32_t i = 0; i < m.n_instruments; ++i) {
            require(m.inst_strike[i] > 0.0,
                    "instruments[" + std::to_string(i) + "]: strike must be > 0");
            require(m.inst_maturity_step[i] >= 1 && m.inst_maturity_step[i] <= m.steps,
                    "instruments[" + std::to_string(i) + "]: maturity_step must be in [1, steps]");
            require(m.inst_kind[i] == LTG_CALL || m.inst_kind[i] == LTG_PUT,
                    "instruments: kind must be call or put");
        }
        // device limits of this build
        require(m.n_s_nodes <= kMaxCols, "GPU build supports at most 8 s-nodes");
        require(nlev <= kMaxLev, "GPU build supports at most 1024 leverage cells");
        require(m.n_instruments <= kMaxInstruments, "GPU build supports at most 256 instruments");
        require(m.steps <= 65535 && (uint64_t)(m.n_t_nodes - 1) * m.n_s_nodes < 65536,
                "GPU build supports at most 65535 steps");

        init_common(c.get(), device);
        c->kind = 0;
        c->steps = m.steps;
        c->cols = m.n_s_nodes;
        c->rows = m.n_t_nodes;
        c->nlev = nlev;
        c->m = m.n_instruments;
        c->M = 5 + nlev;
        c->N = 2 * m.steps;
        c->s0 = m.s0;
        c->mu = m.mu;
        c->dt = m.dt;
        c->x0 = {m.kappa, m.theta, m.xi, m.rho, m.v0};
        c->x0.insert(c->x0.end(), m.leverage, m.leverage + nlev);
        std::vector<double> tn(m.t_nodes, m.t_nodes + m.n_t_nodes);
        std::vector<uint16_t> rowoff(m.steps);
        for (uint32_t k = 0; k < m.steps; ++k)
            rowoff[k] = (uint16_t)(floor_index(tn, (double)k * m.dt) * m.n_s_nodes);
        upload(c->d_rowoff, rowoff);
        upload(c->d_snodes, std::vector<double>(m.s_nodes, m.s_nodes + m.n_s_nodes));
        upload(c->d_strike, std::vector<double>(m.inst_strike, m.inst_strike + m.n_instruments));
        upload(c->d_kind, std::vector<int32_t>(m.inst_kind, m.inst_kind + m.n_instruments));
        build_events(c.get(), std::vector<uint32_t>(m.inst_maturity_step,
                                                     m.inst_maturity_step + m.n_instruments));
        alloc_call_block(c.get());
        cuda_check(cudaDeviceSynchronize(), "init");
    });
    if (rc != LTG_OK) {
        g_create_error = c->err;
        return rc;
    }
    *out = c.release();
    return LTG_OK;
}

int ltg_create_basket(const ltg_basket_model* mdl, int device, ltg_ctx** out) {
    if (!out || !mdl) {
        g_create_error = "null argument";
        return LTG_EINVAL;
    }
    *out = nullptr;
    auto c = std::make_unique<ltg_ctx>();
    const int rc = guarded(c.get(), [&] {
        const ltg_basket_model& m = *mdl;
        require(m.n_assets >= 1 && m.n_assets <= (uint32_t)kMaxAssets,
                "basket: n_assets must be in [1, 16]");
        require(m.s0 && m.chol && m.sigma, "basket: null array");
        require(m.steps > 0, "basket: steps must be > 0");
        require(m.dt > 0.0, "basket: dt must be > 0");
        require(std::isfinite(m.r), "basket: r must be finite");
        require(m.n_instruments > 0 && m.n_instruments <= (uint32_t)kMaxInstruments,
                "basket: 1..256 instruments");
        for (uint32_t a = 0; a < m.n_assets; ++a) {
            require(m.s0[a] > 0.0, "basket: s0 must be > 0");
            for (uint32_t b = 0; b < m.n_assets; ++b)
                require(std::isfinite(m.chol[a * m.n_assets + b]) &&
                            (b <= a || m.chol[a * m.n_assets + b] == 0.0),
                        "basket: chol must be finite and lower-triangular");
        }
        for (uint32_t i = 0; i < m.n_instruments; ++i) {
            require(m.inst_asset[i] < m.n_assets, "basket: instrument asset out of range");
            require(m.inst_strike[i] > 0.0, "basket: strike must be > 0");
            require(m.inst_maturity_step[i] >= 1 && m.inst_maturity_step[i] <= m.steps,
                    "basket: maturity_step must be in [1, steps]");
            require(m.inst_kind[i] == LTG_CALL || m.inst_kind[i] == LTG_PUT,
                    "basket: kind must be call or put");
        }
        init_common(c.get(), device);
        c->kind = 1;
        c->n_assets = m.n_assets;
        c->steps = m.steps;
        c->dt = m.dt;
        c->r = m.r;
        c->m = m.n_instruments;
        c->M = m.n_assets;
        c->N = m.steps * m.n_assets;
        c->chol.assign(m.chol, m.chol + m.n_assets * m.n_assets);
        c->s0v.assign(m.s0, m.s0 + m.n_assets);
        c->x0.assign(m.sigma, m.sigma + m.n_assets);
        upload(c->d_strike, std::vector<double>(m.inst_strike, m.inst_strike + m.n_instruments));
        upload(c->d_kind, std::vector<int32_t>(m.inst_kind, m.inst_kind + m.n_instruments));
        upload(c->d_asset, std::vector<uint32_t>(m.inst_asset, m.inst_asset + m.n_instruments));
        build_events(c.get(), std::vector<uint32_t>(m.inst_maturity_step,
                                                     m.inst_maturity_step + m.n_instruments));
        alloc_call_block(c.get());
        cuda_check(cudaDeviceSynchronize(), "init");
    });
    if (rc != LTG_OK) {
        g_create_error = c->err;
        return rc;
    }
    *out = c.release();
    return LTG_OK;
}


int ltg_create_heston_devices(const ltg_heston_model* model, const int* devices, int n,
                              ltg_ctx** out) {
    return create_group(devices, n, out, [&](int dev, ltg_ctx** m) {
        return ltg_create_heston(model, dev, m);
    });
}

int ltg_create_basket_devices(const ltg_basket_model* model, const int* devices, int n,
                              ltg_ctx** out) {
    return create_group(devices, n, out, [&](int dev, ltg_ctx** m) {
        return ltg_create_basket(model, dev, m);
    });
}

void ltg_destroy(ltg_ctx* ctx) { delete ctx; }

const char* ltg_last_error(const ltg_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

size_t ltg_num_params(const ltg_ctx* ctx) { return ctx ? ctx->M : 0; }
size_t ltg_num_outputs(const ltg_ctx* ctx) { return ctx ? ctx->m : 0; }
size_t ltg_num_randoms(const ltg_ctx* ctx) { return ctx ? ctx->N : 0; }

int ltg_pack_params(const ltg_ctx* ctx, double* x, size_t M) {
    if (!ctx || !x || M != ctx->M) return LTG_EINVAL;
    std::copy(ctx->x0.begin(), ctx->x0.end(), x);
    return LTG_OK;
}

int ltg_rng_exact(const ltg_ctx* ctx) {
    return ctx ? (ctx->h_rc.exact_log && ctx->h_rc.exact_exp) : 0;
}

int ltg_shard_plan(uint64_t paths, int rank, int world, ltg_shard* out) {
    if (!out || world < 1 || rank < 0 || rank >= world || paths == 0) return LTG_EINVAL;
    *out = make_plan(paths, rank, world);
    return LTG_OK;
}

namespace {

// Caller-supplied draws for one call (ltg_*_draws): validates the source as
// the reference does (forward_pass's dimension check, expectation.hpp:156-159;
// BufferDrawSource / SampleSpaceSource's row bound, rng.hpp:160-161,
// expectation.hpp:92-94, raised here before any launch instead of mid-pass),
// uploads this rank's rows (and those of the fresh step-2 path set) and
// releases them when the call ends, so the Philox calls' HBM plan keeps the
// memory.
struct DrawScope {
    ltg_ctx* c = nullptr;
    DrawScope(ltg_ctx* ctx, const ltg_draws* src, const ltg_mc_config& cfg,
              const ltg_shard& plan) {
        if (!src) return;
        require(src->data != nullptr, "null draw buffer");
        require(cfg.precision == LTG_FP64, "caller draws: fp64 only (the reference's arithmetic)");
        require_f(src->dim == ctx->N, [&] {
            return "forward_pass: draw source dimension " + std::to_string(src->dim) +
                   " != tape randoms " + std::to_string(ctx->N);
        });
        require(src->rows <= (uint64_t(1) << 62) / std::max<uint64_t>(1, src->dim),
                "draw buffer size overflows");
        const uint64_t need_rows = cfg.fresh_step2_paths ? 2 * cfg.paths : cfg.paths;
        require_f(src->rows >= need_rows, [&] {
            return "BufferDrawSource: path index out of range (" + std::to_string(need_rows) +
                   " paths need draws, the buffer has " + std::to_string(src->rows) + ")";
        });
        c = ctx;
        const uint64_t rows = plan.path_end - plan.path_begin;
        const uint64_t n_regions = cfg.fresh_step2_paths ? 2 : 1;
        const size_t row_bytes = size_t(ctx->N) * 8;
        const size_t need = std::max<size_t>(8, size_t(rows * n_regions) * row_bytes);
        if (need > ctx->d_draws.bytes) {
            // a previous Philox call's draw store may hold the free HBM
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            if (need + (size_t(1) << 30) > free_b) {
                ctx->d_ztab.release();
                ctx->plan_key.clear();
            }
            ctx->d_draws.ensure(need);
        }
        if (rows) {
            cuda_check(cudaMemcpyAsync(ctx->d_draws.p, src->data + plan.path_begin * ctx->N,
                                       rows * row_bytes, cudaMemcpyHostToDevice, ctx->stream),
                       "H2D draws");
            if (cfg.fresh_step2_paths)
                cuda_check(cudaMemcpyAsync(ctx->d_draws.as<double>() + rows * ctx->N,
                                           src->data + (cfg.paths + plan.path_begin) * ctx->N,
                                           rows * row_bytes, cudaMemcpyHostToDevice, ctx->stream),
                           "H2D draws");
        }
        ctx->draws_on = true;
        ctx->draws_rowsA = rows;
        ctx->draws_row0A = plan.path_begin;
        ctx->draws_row0B = cfg.paths + plan.path_begin;
    }
    ~DrawScope() {
        if (!c) return;
        c->draws_on = false;
        cudaStreamSynchronize(c->stream);
        c->d_draws.release();
    }
};

int gradient_impl(ltg_ctx* ctx, const double* x, size_t M, const double* targets, size_t m,
                  const ltg_mc_config* cfg, ltg_report* report, bool tangent,
                  const ltg_draws* src = nullptr) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx)) {
        const ltg_report proto = report ? *report : ltg_report{};
        return group_run(ctx, [&](ltg_ctx* mb, size_t i) {
            if (i == 0) return gradient_impl(mb, x, M, targets, m, cfg, report, tangent, src);
            // the other ranks' identical reports land in scratch (same nullness,
            // so every member validates alike)
            std::vector<double> means(ctx->m), lambda(ctx->m), grad(ctx->M), se(ctx->m);
            ltg_report r = proto;
            r.means = proto.means ? means.data() : nullptr;
            r.lambda = proto.lambda ? lambda.data() : nullptr;
            r.grad = proto.grad ? grad.data() : nullptr;
            r.std_errors = proto.std_errors ? se.data() : nullptr;
            return gradient_impl(mb, x, M, targets, m, cfg, report ? &r : nullptr, tangent, src);
        });
    }
    return guarded(ctx, [&] {
        validate_cfg(ctx, cfg, M);
        require(x && targets && report && report->means && report->lambda && report->grad,
                "null buffer");
        require_f(m == ctx->m, [&] {
            return "gradient_of_G: " + std::to_string(m) + " targets for " +
                   std::to_string(ctx->m) + " outputs";
        });
        require(!(cfg->memory_mode == LTG_MODE_STORE && cfg->fresh_step2_paths),
                "gradient_of_G: fresh_step2_paths replays nothing, so stored forward state "
                "cannot be used; switch to recompute mode");
        if (tangent)
            require(ctx->kind == 0 && cfg->precision == LTG_FP64 &&
                        heston_tangent_supported(ctx->cols, ctx->nlev),
                    "gradient_of_G_tangent: fp64 Heston models with one leverage column and at "
                    "most 4 leverage rows (M <= 9); use ltg_gradient_of_G");
        check_params(ctx, x);
        const ltg_shard plan = make_plan(cfg->paths, ctx->rank, ctx->world);
        const DrawScope draws(ctx, src, *cfg, plan);
        // fp32 gradients are specified where the variance process stays off
        // the truncation kink, i.e. under the Feller condition 2*kappa*theta
        // >= xi^2 (configs 1-3/5, including the local-vol embeddings with
        // kappa = xi = 0). Below it, V sits at max(V, 0)'s kink on many paths,
        // where sqrt's pathwise derivative 0.5/sqrt(V) turns fp32 rounding of
        // V into O(1) adjoint noise: refused, not approximated.
        if (ctx->fp32 && ctx->kind == 0)
            require(2.0 * x[0] * x[1] >= x[2] * x[2],
                    "fp32 gradient_of_G needs the Feller condition 2*kappa*theta >= xi^2 "
                    "(its accuracy bar is not met at the variance truncation kink); use fp64");
        const uint32_t nm = ctx->m;
        // one pinned staging area per call: [x | targets] in, then the report
        // and the rare flag out (sized up front: a graph captures its address)
        const size_t base = ctx->M + nm;
        double* st = ctx->stage(base + out_doubles(ctx) + 1);
        double* out = st + base;
        // lean call (one GPU, no collective): the kernels read [x | targets]
        // from the staging area, the last reduction writes the report back
        // into it and clears the rare flag, so the call's device work is its
        // kernels alone — no H2D / D2H copy, no flag memset
        const bool lean = !src && !ctx->comm && !ctx->loop && ctx->world == 1;
        const bool graphable = lean && !cfg->fresh_step2_paths;
        struct PubScope {
            ltg_ctx* c;
            ~PubScope() { c->pub = nullptr; }
        } pub_scope{ctx};
        ctx->pub = lean ? out : nullptr;
        const std::string key = std::string(tangent ? "tangent" : "grad") + "/" +
                                std::to_string(cfg->paths) + "/" + std::to_string(cfg->antithetic) +
                                "/" + std::to_string(cfg->precision);
        // (caller draws run the exact slow paths from the start: DrawScope)
        for (ctx->safe = src ? 1 : start_safe(ctx);; ctx->safe = 1) {
            const uint32_t rerun = ctx->safe && !src && !start_safe(ctx) ? 1u : 0u;
            ctx->timing = ltg_timing{};
            ctx->timing_pending = 0;
            ctx->timing.safe_rerun = rerun;
            run_body(ctx, graphable && !ctx->safe, key, [&] {
                upload_x(ctx, x, targets);
                if (!lean || !ctx->flag_clean) reset_flags(ctx);
                if (tangent) {
                    if (cfg->fresh_step2_paths) {
                        run_pass1(ctx, *cfg, plan, true, false);
                        run_tangent(ctx, *cfg, plan, false);
                    } else {
                        run_tangent(ctx, *cfg, plan, true);
                    }
                } else {
                    const bool ckpt = run_pass1(ctx, *cfg, plan, true, !cfg->fresh_step2_paths);
                    run_pass2(ctx, *cfg, plan, ckpt, true);
                }
                if (!lean) copy_out(ctx, out);
            });
            const bool rare = wait_rare(ctx, out + out_doubles(ctx));
            if (lean) ctx->flag_clean = true;  // (the last reduction cleared it)
            if (!rare || ctx->safe) break;
        }
        ctx->safe = 0;
        ctx->timing_pending = 1;  // event times read on demand (settle_timing)
        report->G = out[0];
        std::memcpy(report->means, out + 1, nm * 8);
        if (report->std_errors) std::memcpy(report->std_errors, out + 1 + nm, nm * 8);
        std::memcpy(report->lambda, out + 1 + 2 * nm, nm * 8);
        std::memcpy(report->grad, out + 1 + 3 * nm, ctx->M * 8);
        report->paths = cfg->paths;
        report->seed = cfg->seed;
        report->mode = cfg->memory_mode;
    });
}

}  // namespace

int ltg_gradient_of_G(ltg_ctx* ctx, const double* x, size_t M, const double* targets, size_t m,
                      const ltg_mc_config* cfg, ltg_report* report) {
    return gradient_impl(ctx, x, M, targets, m, cfg, report, false);
}

int ltg_gradient_of_G_tangent(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                              size_t m, const ltg_mc_config* cfg, ltg_report* report) {
    return gradient_impl(ctx, x, M, targets, m, cfg, report, true);
}

int ltg_gradient_of_G_draws(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                            size_t m, const ltg_draws* src, const ltg_mc_config* cfg,
                            ltg_report* report) {
    if (!src) {
        if (ctx && !is_group(ctx)) ctx->err = "null draw source";
        return LTG_EINVAL;
    }
    return gradient_impl(ctx, x, M, targets, m, cfg, report, false, src);
}

int ltg_chunk_sums(ltg_ctx* ctx, const double* x, size_t M, const double* lambda, size_t m,
                   uint64_t seed, int antithetic, uint64_t path0, uint64_t npaths,
                   double* sums, double* sumsq, double* adjoint) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_solo(ctx, [&](ltg_ctx* mb) {
            return ltg_chunk_sums(mb, x, M, lambda, m, seed, antithetic, path0, npaths, sums,
                                  sumsq, adjoint);
        });
    return guarded(ctx, [&] {
        require(x && lambda && sums && sumsq && adjoint, "null buffer");
        require(M == ctx->M && m == ctx->m, "chunk_sums: size mismatch");
        require(npaths > 0, "chunk_sums: paths must be > 0");
        check_params(ctx, x);
        ltg_mc_config cfg{npaths, seed, antithetic, 0, 0, LTG_FP64};
        const ltg_shard plan = make_plan(npaths, 0, 1);
        ctx->stage(std::max<size_t>(M + m, 2 * m + M + 1));  // (no reallocation mid-call)
        struct Reset {
            ltg_ctx* c;
            ~Reset() { c->path_base = 0; }
        } reset{ctx};
        for (ctx->safe = start_safe(ctx);; ctx->safe = 1) {
            const uint32_t rerun = ctx->safe && !start_safe(ctx) ? 1u : 0u;
            ctx->timing = ltg_timing{};
            ctx->timing_pending = 0;
            ctx->timing.safe_rerun = rerun;
            ctx->path_base = path0;
            upload_x(ctx, x, nullptr);
            reset_flags(ctx);
            const bool ckpt = run_pass1(ctx, cfg, plan, false, true);
            // pass 2 seeded with the caller's lambda instead of pass 1's
            cuda_check(cudaMemcpyAsync(ctx->d_res.as<double>() + 1 + 2 * ctx->m, lambda, m * 8,
                                       cudaMemcpyHostToDevice, ctx->stream),
                       "H2D");
            run_pass2(ctx, cfg, plan, ckpt);
            double* st = ctx->stage(2 * m + M + 1);
            cuda_check(cudaMemcpyAsync(st, ctx->d_tot1.p, 2 * m * 8, cudaMemcpyDeviceToHost,
                                       ctx->stream),
                       "D2H");
            cuda_check(cudaMemcpyAsync(st + 2 * m, ctx->d_tot2.p, M * 8, cudaMemcpyDeviceToHost,
                                       ctx->stream),
                       "D2H");
            copy_rare(ctx, st + 2 * m + M);
            if (!wait_rare(ctx, st + 2 * m + M) || ctx->safe) {
                std::memcpy(sums, st, m * 8);
                std::memcpy(sumsq, st + m, m * 8);
                std::memcpy(adjoint, st + 2 * m, M * 8);
                break;
            }
        }
        ctx->safe = 0;
    });
}

namespace {

int means_impl(ltg_ctx* ctx, const double* x, size_t M, const ltg_mc_config* cfg,
               double* means, double* std_errors, const ltg_draws* src) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_run(ctx, [&](ltg_ctx* mb, size_t i) {
            if (i == 0) return means_impl(mb, x, M, cfg, means, std_errors, src);
            std::vector<double> mv(ctx->m), sv(ctx->m);
            return means_impl(mb, x, M, cfg, means ? mv.data() : nullptr,
                              std_errors ? sv.data() : nullptr, src);
        });
    return guarded(ctx, [&] {
        validate_cfg(ctx, cfg, M);
        require(x && means, "null buffer");
        check_params(ctx, x);
        const ltg_shard plan = make_plan(cfg->paths, ctx->rank, ctx->world);
        const DrawScope draws(ctx, src, *cfg, plan);
        const uint32_t nm = ctx->m;
        // staging: [x] in, the report and the rare flag out (as gradient_impl)
        const size_t base = ctx->M;
        double* st = ctx->stage(base + out_doubles(ctx) + 1);
        double* out = st + base;
        const bool lean = !src && !ctx->comm && !ctx->loop && ctx->world == 1;
        const bool graphable = lean;
        struct PubScope {
            ltg_ctx* c;
            ~PubScope() { c->pub = nullptr; }
        } pub_scope{ctx};
        ctx->pub = lean ? out : nullptr;
        const std::string key = "means/" + std::to_string(cfg->paths) + "/" +
                                std::to_string(cfg->antithetic) + "/" +
                                std::to_string(cfg->precision);
        // (caller draws run the exact slow paths from the start: DrawScope)
        for (ctx->safe = src ? 1 : start_safe(ctx);; ctx->safe = 1) {
            const uint32_t rerun = ctx->safe && !src && !start_safe(ctx) ? 1u : 0u;
            ctx->timing = ltg_timing{};
            ctx->timing_pending = 0;
            ctx->timing.safe_rerun = rerun;
            run_body(ctx, graphable && !ctx->safe, key, [&] {
                upload_x(ctx, x, nullptr);
                if (!lean || !ctx->flag_clean) reset_flags(ctx);
                run_pass1(ctx, *cfg, plan, false, false, true);
                if (!lean) copy_out(ctx, out);
            });
            const bool rare = wait_rare(ctx, out + out_doubles(ctx));
            if (lean) ctx->flag_clean = true;
            if (!rare || ctx->safe) break;
        }
        ctx->safe = 0;
        ctx->timing_pending = 2;
        std::memcpy(means, out + 1, nm * 8);
        if (std_errors) std::memcpy(std_errors, out + 1 + nm, nm * 8);
    });
}

}  // namespace

int ltg_estimate_means(ltg_ctx* ctx, const double* x, size_t M, const ltg_mc_config* cfg,
                       double* means, double* std_errors) {
    return means_impl(ctx, x, M, cfg, means, std_errors, nullptr);
}

int ltg_estimate_means_draws(ltg_ctx* ctx, const double* x, size_t M, const ltg_draws* src,
                             uint64_t paths, double* means, double* std_errors) {
    if (!src) {
        if (ctx && !is_group(ctx)) ctx->err = "null draw source";
        return LTG_EINVAL;
    }
    // estimate_means(Kernel, params, PathDrawSource, paths, workers): fp64, no
    // seed or antithetic pairing (the source fixes the draws)
    const ltg_mc_config cfg{paths, 0, 0, 0, LTG_MODE_RECOMPUTE, LTG_FP64};
    return means_impl(ctx, x, M, &cfg, means, std_errors, src);
}

int ltg_finite_diff_gradient_of_G(ltg_ctx* ctx, const double* x, size_t M, const double* targets,
                                  size_t m, const ltg_mc_config* cfg, double h, double* grad) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_run(ctx, [&](ltg_ctx* mb, size_t i) {
            if (i == 0) return ltg_finite_diff_gradient_of_G(mb, x, M, targets, m, cfg, h, grad);
            std::vector<double> g(ctx->M);
            return ltg_finite_diff_gradient_of_G(mb, x, M, targets, m, cfg, h,
                                                 grad ? g.data() : nullptr);
        });
    if (!(h > 0.0)) {
        ctx->err = "finite_diff_gradient_of_G: h must be > 0";
        return LTG_EINVAL;
    }
    if (!x || !targets || !grad || M != ctx->M || m != ctx->m) {
        ctx->err = "finite_diff_gradient_of_G: size mismatch";
        return LTG_EINVAL;
    }
    // expectation.hpp:372-400: central differences of G under common random numbers
    std::vector<double> xv(x, x + M), means(m);
    auto G_at = [&](double& out) {
        const int rc = ltg_estimate_means(ctx, xv.data(), M, cfg, means.data(), nullptr);
        if (rc) return rc;
        double g = 0.0;
        for (size_t o = 0; o < m; ++o) {
            const double l = means[o] - targets[o];
            g += 0.5 * l * l;
        }
        out = g;
        return 0;
    };
    for (size_t j = 0; j < M; ++j) {
        const double saved = xv[j];
        double up = 0, down = 0;
        xv[j] = saved + h;
        int rc = G_at(up);
        if (rc) return rc;
        xv[j] = saved - h;
        rc = G_at(down);
        if (rc) return rc;
        xv[j] = saved;
        grad[j] = (up - down) / (2.0 * h);
    }
    return LTG_OK;
}

int ltg_fill_normals(ltg_ctx* ctx, uint64_t seed, size_t dim, int antithetic, uint64_t path0,
                     uint64_t npaths, double* out) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_solo(ctx, [&](ltg_ctx* mb) {
            return ltg_fill_normals(mb, seed, dim, antithetic, path0, npaths, out);
        });
    return guarded(ctx, [&] {
        require(out != nullptr, "null buffer");
        require(dim > 0 && dim < (size_t(1) << 30), "dimension out of range");
        const size_t n = size_t(npaths) * dim;
        if (n == 0) return;
        ctx->d_normals.ensure(n * 8);
        cuda_check(launch_fill_normals(ctx->d_tab.as<RngTables>(), ctx->h_rc, (uint32_t)seed,
                                       (uint32_t)(seed >> 32), antithetic, path0, npaths,
                                       (uint32_t)dim, ctx->d_normals.as<double>(), ctx->stream),
                   "fill_normals");
        cuda_check(cudaMemcpyAsync(out, ctx->d_normals.p, n * 8, cudaMemcpyDeviceToHost,
                                   ctx->stream),
                   "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "fill_normals");
    });
}

int ltg_inverse_normal(ltg_ctx* ctx, const double* p, size_t n, double* z) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_solo(ctx, [&](ltg_ctx* mb) { return ltg_inverse_normal(mb, p, n, z); });
    return guarded(ctx, [&] {
        require(p && z, "null buffer");
        if (n == 0) return;
        for (size_t i = 0; i < n; ++i)  // rng.hpp:46 throws outside (0, 1)
            require(p[i] > 0.0 && p[i] < 1.0, "inverse_normal_cdf: p outside (0,1)");
        ctx->d_normals.ensure(2 * n * 8);
        double* d_p = ctx->d_normals.as<double>();
        cuda_check(cudaMemcpyAsync(d_p, p, n * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        cuda_check(launch_inverse_normal(ctx->d_tab.as<RngTables>(), ctx->h_rc, d_p, n, d_p + n,
                                         ctx->stream),
                   "inverse_normal");
        cuda_check(cudaMemcpyAsync(z, d_p + n, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "inverse_normal");
    });
}

int ltg_path_payoffs(ltg_ctx* ctx, const double* x, size_t M, uint64_t seed, int antithetic,
                     uint64_t path0, uint64_t npaths, double* y) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx))
        return group_solo(ctx, [&](ltg_ctx* mb) {
            return ltg_path_payoffs(mb, x, M, seed, antithetic, path0, npaths, y);
        });
    return guarded(ctx, [&] {
        require(x && y && M == ctx->M, "path_payoffs: size mismatch");
        check_params(ctx, x);
        if (npaths == 0) return;
        upload_x(ctx, x, nullptr);
        ltg_mc_config cfg{npaths, seed, antithetic, 0, 0, LTG_FP64};
        ltg_shard plan{};
        plan.chunk_paths = kBlock;
        plan.n_chunks = (npaths + kBlock - 1) / kBlock;
        plan.chunk_begin = 0;
        plan.chunk_end = plan.n_chunks;
        Work w = base_work(ctx, cfg, plan);
        w.path_offset = path0;
        w.ckpt_path0 = 0;
        ctx->seg_steps = 16;
        ctx->d_part1.ensure(plan.n_chunks * 2 * ctx->m * 8);
        ctx->d_normals.ensure(npaths * ctx->m * 8);
        if (ctx->kind == 0) {
            ctx->fp32 = 0;
            HestonArgs a = heston_args(ctx, ctx->h_x.data());
            a.partials = ctx->d_part1.as<double>();
            a.path_out = ctx->d_normals.as<double>();
            a.write_sums = 1;
            a.write_ckpt = 0;
            a.safe = 1;  // diagnostic entry: exact slow paths throughout
            cuda_check(launch_heston_pass1(a, w, 0, ctx->stream), "path payoffs");
        } else {
            BasketArgs b = basket_args(ctx, ctx->h_x.data());
            b.partials = ctx->d_part1.as<double>();
            b.path_out = ctx->d_normals.as<double>();
            b.write_sums = 1;
            cuda_check(launch_basket_pass1(b, w, 0, ctx->stream), "path payoffs");
        }
        cuda_check(cudaMemcpyAsync(y, ctx->d_normals.p, npaths * ctx->m * 8,
                                   cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "path payoffs");
    });
}

int ltg_set_hbm_budget(ltg_ctx* ctx, uint64_t bytes) {
    if (!ctx) return LTG_EINVAL;
    ctx->hbm_budget = bytes;
    for (auto& m : ctx->members) m->hbm_budget = bytes;
    return LTG_OK;
}

int ltg_set_timing(ltg_ctx* ctx, int on) {
    if (!ctx) return LTG_EINVAL;
    ctx->timing_on = on != 0;
    for (auto& mb : ctx->members) mb->timing_on = on != 0;
    return LTG_OK;
}

int ltg_last_timing(const ltg_ctx* ctx, ltg_timing* out) {
    if (!ctx || !out) return LTG_EINVAL;
    if (ctx->ready && ctx->timing_pending) {
        cudaSetDevice(ctx->device);
        settle_timing(const_cast<ltg_ctx*>(ctx));
    }
    *out = ctx->timing;
    return LTG_OK;
}

int ltg_nccl_unique_id(unsigned char id[128]) {
    std::string why;
    if (!nccl().load(why)) {
        g_create_error = why;
        return LTG_ECUDA;
    }
    ncclUniqueId u;
    const ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) {
        g_create_error = nccl().GetErrorString(r);
        return LTG_ECUDA;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return LTG_OK;
}

int ltg_attach_nccl(ltg_ctx* ctx, const unsigned char id[128], int rank, int world) {
    if (!ctx) return LTG_EINVAL;
    if (is_group(ctx)) {
        ctx->err = "attach_nccl: a multi-device context has its communicators already";
        return LTG_EINVAL;
    }
    return guarded(ctx, [&] {
        require(id != nullptr && world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        std::string why;
        if (!nccl().load(why)) throw Failure(LTG_ECUDA, why);
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        if (ctx->comm) nccl().CommDestroy(ctx->comm);
        ctx->comm = nullptr;
        ctx->rank = 0;  // single-GPU until the new communicator exists
        ctx->world = 1;
        ncclComm_t comm = nullptr;
        const ncclResult_t r = nccl().CommInitRank(&comm, world, u, rank);
        if (r != ncclSuccess)
            throw Failure(LTG_ECUDA, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
        ctx->comm = comm;
        ctx->rank = rank;
        ctx->world = world;
    });
}

}  // extern "C"
