// basket.cu — gradient_of_G for the config-4 program: n <= 16 correlated
// log-Euler GBMs, constant vols sigma_a as the parameters (the program
// recorded by oracle/ref_driver.cpp record_basket with the reference Tape API).
//
// Forward, per step k and asset a, operation for operation as recorded:
//   w_a = ((L[a][0] z_0 + L[a][1] z_1) + ...) + L[a][a] z_a
//   S_a = S_a * exp(drift_a + vol_a * w_a),
//   drift_a = (r - 0.5 (sigma_a sigma_a)) dt,  vol_a = sigma_a sqrt(dt)
// with draw slot k*n + a of PhiloxNormalSource (rng.hpp:113-127).
//
// Adjoint. The reverse of S' = S exp(x) leaves u = S̄·S unchanged and gives
// x̄ = u, so between two maturities the reverse sweep of every step feeds the
// same u_a into drift̄_a += u_a and vol̄_a += u_a w_{a,k}. Summed in reverse
// order it telescopes to, for each instrument i on asset a maturing at ms:
//   sigmā_a += lambda_i sgn_i 1{payoff_i > 0} S_a(ms) (sqrt(dt) W_a(ms) - sigma_a dt ms),
//   W_a(ms) = sum_{k < ms} w_{a,k}
// (tape.hpp:344-413 applied to the recorded nodes; the tape's own
// accumulation order differs only by rounding). Pass 1 therefore stores
// (S_a, W_a) at each maturity in HBM (the reference's store mode, with 2n
// doubles per path instead of the tape's ~24k nodes), and pass 2 is a short
// streaming epilogue; without room for the store, pass 2 re-simulates the
// paths (recompute mode) and evaluates the same epilogue on the fly.
#include <cuda_runtime.h>

#include "finish.cuh"
#include "kernels.h"
#include "launch_config.h"
#include "rng.cuh"

namespace ltg {
namespace {

constexpr int NA = kMaxAssets;
constexpr int BGS = 16;  // Philox pairs per normal batch (two steps of 16 assets)
#ifndef LTG_BASKET_FUSED
#define LTG_BASKET_FUSED LTG_F64_FUSED  // gen_segment's phases A and B fused (rng.cuh)
#endif
#ifndef LTG_BPB
#define LTG_BPB 8  // central slots evaluated together (measured on config 4)
#endif

__device__ __forceinline__ double warp_sum_b(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// S[a] for a warp-uniform runtime a
__device__ __forceinline__ double pick(const double (&v)[NA], uint32_t a) {
    double r = v[0];
#pragma unroll
    for (int c = 1; c < NA; ++c)
        if (a == (uint32_t)c) r = v[c];
    return r;
}

struct BSmem {
    RngTables* tab;
    double* strike;   // maturity-sorted position
    int* kind;
    int* asset;
    int* inst_id;
    double* lambda;
    double* acc;      // [kWarps][width]
    double* zbuf;     // [2*BGS][kBlock]
    uint16_t* list;   // [kWarps][64*BGS]
};

__host__ __device__ inline size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline size_t basket_smem(uint32_t m, uint32_t width) {
    return al16(sizeof(RngTables)) + al16(m * 8) + 3 * al16(m * 4) + al16(m * 8) +
           al16(size_t(kWarps) * width * 8) + al16(size_t(2 * BGS) * kBlock * 8) +
           al16(size_t(kWarps) * 64 * BGS * 2);
}

__device__ inline BSmem bcarve(char* base, uint32_t m, uint32_t width) {
    BSmem s;
    size_t o = 0;
    auto take = [&](size_t b) {
        char* p = base + o;
        o += al16(b);
        return p;
    };
    s.tab = reinterpret_cast<RngTables*>(take(sizeof(RngTables)));
    s.strike = reinterpret_cast<double*>(take(m * 8));
    s.kind = reinterpret_cast<int*>(take(m * 4));
    s.asset = reinterpret_cast<int*>(take(m * 4));
    s.inst_id = reinterpret_cast<int*>(take(m * 4));
    s.lambda = reinterpret_cast<double*>(take(m * 8));
    s.acc = reinterpret_cast<double*>(take(size_t(kWarps) * width * 8));
    s.zbuf = reinterpret_cast<double*>(take(size_t(2 * BGS) * kBlock * 8));
    s.list = reinterpret_cast<uint16_t*>(take(size_t(kWarps) * 64 * BGS * 2));
    return s;
}

__device__ inline void bload(const BasketArgs& a, const BSmem& s, uint32_t width, bool pass2) {
    load_tables(s.tab, a.tables);
    for (uint32_t i = threadIdx.x; i < a.m; i += kBlock) {
        const uint32_t id = a.inst_order[i];
        s.strike[i] = a.strike[id];
        s.kind[i] = a.kind[id];
        s.asset[i] = (int)a.asset[id];
        s.inst_id[i] = (int)id;
        s.lambda[i] = pass2 ? a.lambda[id] : 0.0;
    }
    for (uint32_t i = threadIdx.x; i < kWarps * width; i += kBlock) s.acc[i] = 0.0;
}

__device__ inline uint64_t bnext_chunk(const Work& w, uint32_t* slot) {
    __syncthreads();
    if (threadIdx.x == 0) {  // (self-resetting counter: heston.cu next_chunk)
        const uint32_t t = atomicAdd(w.counter, 1u);
        if ((uint64_t)t == w.n_chunks + gridDim.x - 1) atomicExch(w.counter, 0u);
        *slot = t;
    }
    __syncthreads();
    return *slot;
}

template <typename Map>
__device__ inline void bflush(double* acc, uint32_t width, double* row, Map map) {
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < width; t += kBlock) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            s += acc[w * width + t];
            acc[w * width + t] = 0.0;
        }
        row[map(t)] = s;
    }
    __syncthreads();
}

// One forward path: S (and W when tracked); at every maturity event `visit`
// is called with the event index. SAFE = false uses glibc exp's main path
// without the |x| >= 512 guard and raises the path's rare flag instead (the
// host then reruns the call with SAFE = true; see heston.cu heston_step).
template <bool TRACK_W, bool SAFE, int NAT, bool DRAWS, typename Visit>
__device__ __forceinline__ void simulate(const BasketArgs& a, const BSmem& s, const Work& w,
                                         uint64_t base, bool neg, const double* drow, bool valid,
                                         double (&S)[NA], double (&W)[NA], unsigned& chk,
                                         Visit visit) {
    const int tid = threadIdx.x, warp = tid >> 5;
    double* zb = s.zbuf + tid;
    uint16_t* wl = s.list + warp * 64 * BGS;
    const uint32_t n = NAT ? (uint32_t)NAT : a.n;  // NAT: asset count fixed at compile time
#pragma unroll
    for (int c = 0; c < NA; ++c) {
        S[c] = a.s0[c];
        W[c] = 0.0;
    }
    uint32_t ev = 0;
    uint32_t ev_step = a.n_events ? a.events[0].step : 0xffffffffu;
    for (uint32_t k0 = 0; k0 < a.steps; k0 += 2) {
        const uint32_t nb = min(2u, a.steps - k0);
        const uint32_t pair0 = (k0 * n) >> 1;
        const int npairs = (int)((nb * n + 1) >> 1);
        if (DRAWS)  // caller draws: slots [k0*n, k0*n + 2*npairs) of the path's row
            copy_draws<double>(drow, valid, 2 * pair0, 2 * npairs, a.steps * n, zb);
        else
            gen_segment<BGS, LTG_BPB, (LTG_BASKET_FUSED != 0)>(base, neg, pair0, npairs,
                                                               w.rk, zb, wl,
                                                               *s.tab, a.rc);
        for (uint32_t j = 0; j < nb; ++j) {
            const uint32_t k = k0 + j;
            double z[NA];
#pragma unroll
            for (int b = 0; b < NA; ++b) z[b] = (uint32_t)b < n ? zb[(j * n + b) * kBlock] : 0.0;
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                if ((uint32_t)c < n) {
                    double wc = __dmul_rn(a.chol[c * NA + 0], z[0]);
#pragma unroll
                    for (int b = 1; b <= c; ++b)
                        wc = __dadd_rn(wc, __dmul_rn(a.chol[c * NA + b], z[b]));
                    if (TRACK_W) W[c] += wc;
                    const double x = __dadd_rn(a.drift[c], __dmul_rn(a.vol[c], wc));
                    double E;
                    if (SAFE) {
                        E = exp_ref(x, s.tab->exp_tab, a.rc);
                    } else {
                        // |x| >= 512 <=> (hi & 0x7ff00000) >= 0x40800000 (flag threshold
                        // 0x7ca00000 after the shift, as in heston.cu)
                        chk = max(chk, ((unsigned)__double2hiint(x) & 0x7ff00000u) + 0x3c200000u);
                        E = glibc_exp_main(x, s.tab->exp_tab, a.rc);  // validated table
                    }
                    S[c] = __dmul_rn(S[c], E);
                }
            }
            if (k + 1 == ev_step) {
                visit(ev, k + 1);
                ++ev;
                ev_step = ev < a.n_events ? a.events[ev].step : 0xffffffffu;
            }
        }
    }
}

constexpr unsigned kBRareThr = 0x7ca00000u;

// NAT = 16 (config 4) specialises the asset loops; NAT = 0 takes a.n at run time
template <bool SAFE, int NAT, bool DRAWS = false>
__global__ void __launch_bounds__(kBlock, 4) basket_pass1_kernel(BasketArgs a, Work w) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ uint32_t chunk_slot;
    const uint32_t m = a.m, width = 2 * m, n = NAT ? (uint32_t)NAT : a.n;
    const BSmem s = bcarve(smem_raw, m, width);
    bload(a, s, width, false);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* acc = s.acc + warp * width;
    for (uint64_t ci = bnext_chunk(w, &chunk_slot); ci < w.n_chunks;
         ci = bnext_chunk(w, &chunk_slot)) {
        const uint64_t chunk = w.chunk_begin + ci;
        for (uint64_t r0 = 0; r0 < w.chunk_paths; r0 += kBlock) {
            const uint64_t gp = chunk * w.chunk_paths + r0 + tid;
            const bool valid = gp < w.paths;
            const uint64_t path = w.path_offset + gp;
            const uint64_t base = w.antithetic ? path >> 1 : path;
            const bool neg = w.antithetic && (path & 1u);
            double S[NA], W[NA];
            unsigned chk = 0;
            auto visit = [&](uint32_t ev, uint32_t ms) {
                const MaturityEvent e = a.events[ev];
                if (a.write_store && valid) {
#pragma unroll
                    for (int c = 0; c < NA; ++c)
                        if ((uint32_t)c < n)
                            a.store[((uint64_t)ev * n + c) * a.store_stride +
                                    (gp - w.ckpt_path0)] = make_double2(S[c], W[c]);
                }
                if (!a.write_sums) return;
                for (uint32_t pos = e.begin; pos < e.end; ++pos) {
                    const double Sa = pick(S, (uint32_t)s.asset[pos]);
                    const double K = s.strike[pos];
                    const double d = s.kind[pos] == 1 ? __dsub_rn(K, Sa) : __dsub_rn(Sa, K);
                    const double y = (valid && d > 0.0) ? d : 0.0;
                    if (a.path_out && valid)
                        a.path_out[(gp - w.ckpt_path0) * m + s.inst_id[pos]] = y;
                    const double s1 = warp_sum_b(y);
                    const double s2 = warp_sum_b(__dmul_rn(y, y));
                    if (lane == 0) {
                        acc[pos] += s1;
                        acc[m + pos] += s2;
                    }
                }
            };
            const double* drow = DRAWS ? a.draws + (base - a.draws_row0) * ((uint64_t)a.steps * n)
                                       : nullptr;
            if (a.write_store)
                simulate<true, SAFE, NAT, DRAWS>(a, s, w, base, neg, drow, valid, S, W, chk, visit);
            else
                simulate<false, SAFE, NAT, DRAWS>(a, s, w, base, neg, drow, valid, S, W, chk,
                                                  visit);
            if (chk >= kBRareThr && valid) atomicOr(a.rare, 1u);
        }
        if (a.write_sums) {
            double* row = a.partials + ci * width;
            bflush(s.acc, width, row, [&](uint32_t t) {
                return t < m ? (uint32_t)s.inst_id[t] : m + (uint32_t)s.inst_id[t - m];
            });
        }
    }
    if (w.fuse) fused_tail(a.partials, w.n_chunks, width, w);
}

// sigmā contribution of instrument `pos` observed at maturity ms
__device__ __forceinline__ double contribution(const BasketArgs& a, const BSmem& s, uint32_t pos,
                                               uint32_t ms, double Sa, double Wa) {
    const uint32_t c = (uint32_t)s.asset[pos];
    const double K = s.strike[pos];
    const bool put = s.kind[pos] == 1;
    const double d = put ? K - Sa : Sa - K;
    if (!(d > 0.0)) return 0.0;
    const double lam = put ? -s.lambda[pos] : s.lambda[pos];
    return lam * Sa * (a.sqdt * Wa - a.sigma[c] * a.dt * (double)ms);
}

template <bool SAFE, int NAT, bool DRAWS = false>
__global__ void __launch_bounds__(kBlock, 4) basket_pass2_kernel(BasketArgs a, Work w) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ uint32_t chunk_slot;
    const uint32_t m = a.m, n = NAT ? (uint32_t)NAT : a.n, width = n;
    const BSmem s = bcarve(smem_raw, m, width);
    bload(a, s, width, true);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* acc = s.acc + warp * width;
    for (uint64_t ci = bnext_chunk(w, &chunk_slot); ci < w.n_chunks;
         ci = bnext_chunk(w, &chunk_slot)) {
        const uint64_t chunk = w.chunk_begin + ci;
        for (uint64_t r0 = 0; r0 < w.chunk_paths; r0 += kBlock) {
            const uint64_t gp = chunk * w.chunk_paths + r0 + tid;
            const bool valid = gp < w.paths;
            auto add = [&](uint32_t pos, double v) {
                const double t = warp_sum_b(valid ? v : 0.0);
                if (lane == 0) acc[s.asset[pos]] += t;
            };
            if (a.use_store) {
                for (uint32_t ev = 0; ev < a.n_events; ++ev) {
                    const MaturityEvent e = a.events[ev];
                    for (uint32_t pos = e.begin; pos < e.end; ++pos) {
                        double2 sw = make_double2(1.0, 0.0);
                        if (valid)
                            sw = a.store[((uint64_t)ev * n + s.asset[pos]) * a.store_stride +
                                         (gp - w.ckpt_path0)];
                        add(pos, contribution(a, s, pos, e.step, sw.x, sw.y));
                    }
                }
            } else {
                const uint64_t path = w.path_offset + gp;
                const uint64_t base = w.antithetic ? path >> 1 : path;
                const bool neg = w.antithetic && (path & 1u);
                double S[NA], W[NA];
                unsigned chk = 0;
                const double* drow =
                    DRAWS ? a.draws + (base - a.draws_row0) * ((uint64_t)a.steps * n) : nullptr;
                simulate<true, SAFE, NAT, DRAWS>(a, s, w, base, neg, drow, valid, S, W, chk,
                                     [&](uint32_t ev, uint32_t ms) {
                    const MaturityEvent e = a.events[ev];
                    for (uint32_t pos = e.begin; pos < e.end; ++pos) {
                        const uint32_t c = (uint32_t)s.asset[pos];
                        add(pos, contribution(a, s, pos, ms, pick(S, c), pick(W, c)));
                    }
                });
                if (chk >= kBRareThr && valid) atomicOr(a.rare, 1u);
            }
        }
        double* row = a.partials + ci * width;
        bflush(s.acc, width, row, [](uint32_t t) { return t; });
    }
    if (w.fuse) fused_tail(a.partials, w.n_chunks, width, w);
}

template <typename K>
cudaError_t blaunch(K kernel, const BasketArgs& a, const Work& w, int grid, size_t smem,
                    cudaStream_t st) {
    const int resident = resident_grid((const void*)kernel, smem, kBlock);
    if (grid <= 0) grid = resident;
    if ((uint64_t)grid > w.n_chunks) grid = (int)w.n_chunks;
    if (grid < 1) grid = 1;
    return launch_kernel(kernel, grid, kBlock, smem, st, a, w);
}

}  // namespace

cudaError_t launch_basket_pass1(const BasketArgs& a, const Work& w, int grid, cudaStream_t st) {
    const size_t smem = basket_smem(a.m, 2 * a.m);
    if (a.draws)  // caller draws: exact slow paths only (the host runs safe)
        return !a.safe ? cudaErrorInvalidValue
               : a.n == kMaxAssets
                   ? blaunch(basket_pass1_kernel<true, kMaxAssets, true>, a, w, grid, smem, st)
                   : blaunch(basket_pass1_kernel<true, 0, true>, a, w, grid, smem, st);
    if (a.n == kMaxAssets)
        return a.safe ? blaunch(basket_pass1_kernel<true, kMaxAssets>, a, w, grid, smem, st)
                      : blaunch(basket_pass1_kernel<false, kMaxAssets>, a, w, grid, smem, st);
    return a.safe ? blaunch(basket_pass1_kernel<true, 0>, a, w, grid, smem, st)
                  : blaunch(basket_pass1_kernel<false, 0>, a, w, grid, smem, st);
}

cudaError_t launch_basket_pass2(const BasketArgs& a, const Work& w, int grid, cudaStream_t st) {
    const size_t smem = basket_smem(a.m, a.n);
    if (a.draws)
        return !a.safe ? cudaErrorInvalidValue
               : a.n == kMaxAssets
                   ? blaunch(basket_pass2_kernel<true, kMaxAssets, true>, a, w, grid, smem, st)
                   : blaunch(basket_pass2_kernel<true, 0, true>, a, w, grid, smem, st);
    if (a.n == kMaxAssets)
        return a.safe ? blaunch(basket_pass2_kernel<true, kMaxAssets>, a, w, grid, smem, st)
                      : blaunch(basket_pass2_kernel<false, kMaxAssets>, a, w, grid, smem, st);
    return a.safe ? blaunch(basket_pass2_kernel<true, 0>, a, w, grid, smem, st)
                  : blaunch(basket_pass2_kernel<false, 0>, a, w, grid, smem, st);
}

}  // namespace ltg
