// finish.cuh — the end of a call on the device: means, standard errors,
// lambda and G from pass 1's totals, the gradient from pass 2's, the report
// published to the caller's pinned buffer (reduce_final_kernel, or the last
// CTA of a pass launch with a fused reduction: fused_tail).
#pragma once
#include <cstdint>

#include "kernels.h"

namespace ltg {

// means_from_sums (expectation.hpp:251-269) for output o
__device__ inline void finalize_mean(const double* totals, uint32_t m, uint64_t paths,
                              const Finish& f, double* res, uint32_t o) {
    const double P = (double)paths;
    const double mean = __ddiv_rn(totals[o], P);
    res[1 + o] = mean;
    if (paths > 1) {
        double var = __ddiv_rn(__dsub_rn(totals[m + o], __dmul_rn(__dmul_rn(P, mean), mean)),
                               __dsub_rn(P, 1.0));
        var = var > 0.0 ? var : 0.0;
        res[1 + m + o] = __dsqrt_rn(__ddiv_rn(var, P));
    } else {
        res[1 + m + o] = 0.0;
    }
    if (f.tgt_inline || f.targets)  // lambda (:329-334)
        res[1 + 2 * m + o] = __dsub_rn(mean, f.tgt_inline ? f.tgt_in[o] : f.targets[o]);
}

// Group sums -> totals (ascending group order), then the call's finishing
// step in the same single-CTA launch:
//   means: means, std errors, lambda per output (one thread each), then
//          G = sum_o 0.5 * lambda_o^2 in ascending o (:329-334);
//   grad:  grad = total / P (:340-342);
//   grad_tangent: grad[d] = (sum_i lambda_i * J[i][d]) / P, i ascending,
//          J = totals + 2m, lambda from res (written by `means` above when
//          both are set).
__device__ inline void finish_call(const double* out, const Finish& f) {
    if (!(f.means || f.grad || f.grad_tangent || f.pub)) return;
    __syncthreads();  // out visible to the block
    if (f.means) {
        for (uint32_t o = threadIdx.x; o < f.m; o += blockDim.x)
            finalize_mean(out, f.m, f.paths, f, f.res, o);
        __syncthreads();
        if (threadIdx.x == 0) {
            double G = 0.0;
            if (f.tgt_inline || f.targets) {
                const double* lambda = f.res + 1 + 2 * f.m;
                for (uint32_t o = 0; o < f.m; ++o)
                    G = __dadd_rn(G, __dmul_rn(__dmul_rn(0.5, lambda[o]), lambda[o]));
            }
            f.res[0] = G;
        }
    }
    if (f.grad)
        for (uint32_t j = threadIdx.x; j < f.M; j += blockDim.x)
            f.grad_out[j] = __ddiv_rn(out[j], (double)f.paths);
    if (f.grad_tangent) {
        const double* J = out + 2 * f.m;
        const double* lambda = f.res + 1 + 2 * f.m;
        for (uint32_t d = threadIdx.x; d < f.M; d += blockDim.x) {
            double t = 0.0;
            for (uint32_t i = 0; i < f.m; ++i)
                t = __dadd_rn(t, __dmul_rn(lambda[i], J[(size_t)i * f.M + d]));
            f.grad_out[d] = __ddiv_rn(t, (double)f.paths);
        }
    }
    if (f.pub) {
        __syncthreads();  // this block's writes to res / grad_out are visible to it
        for (uint32_t i = threadIdx.x; i < f.pub_n; i += blockDim.x) f.pub[i] = __ldcg(f.pub_src + i);
        if (threadIdx.x == 0)
            reinterpret_cast<uint32_t*>(f.pub + f.pub_n)[0] = atomicExch(f.rare, 0u);
    }
}

// The fused reduction of a pass launch (Work::fuse, small tables on one GPU):
// the CTA that finishes last reduces the launch's chunk rows [0, n_chunks)
// exactly as launch_reduce_chunks does — each column summed over a group of
// kGroup rows in ascending row order, then over the groups in ascending
// order, every sum starting from 0.0 — and finishes the call. Thread items
// are (group, column) pairs, so the groups' addition chains run in parallel.
// Called by all threads of every CTA after its last chunk row is written.
__device__ inline void fused_tail(const double* table, uint64_t n_chunks, uint32_t width,
                                  const Work& w) {
    __shared__ uint32_t is_last;
    __threadfence();  // every thread's row writes before the CTA's count
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t t = atomicAdd(w.done, 1u);
        is_last = t == gridDim.x - 1 ? 1u : 0u;
        if (is_last) atomicExch(w.done, 0u);  // (left zero for the next launch)
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const uint64_t ng = (n_chunks + kGroup - 1) / kGroup;
    for (uint64_t it = threadIdx.x; it < ng * width; it += blockDim.x) {
        const uint64_t g = it / width;
        const uint32_t col = (uint32_t)(it - g * width);
        const uint64_t r0 = g * kGroup, r1 = min(r0 + (uint64_t)kGroup, n_chunks);
        const double* p = table + r0 * width + col;
        double s = 0.0;
        uint64_t r = r0;
        constexpr int kBatch = 16;  // loads in flight ahead of the ordered additions
        for (; r + kBatch <= r1; r += kBatch, p += kBatch * width) {
            double v[kBatch];
#pragma unroll
            for (int b = 0; b < kBatch; ++b) v[b] = __ldcg(p + b * width);
#pragma unroll
            for (int b = 0; b < kBatch; ++b) s = __dadd_rn(s, v[b]);
        }
        for (; r < r1; ++r, p += width) s = __dadd_rn(s, __ldcg(p));
        w.groups[g * width + col] = s;
    }
    __syncthreads();
    for (uint32_t col = threadIdx.x; col < width; col += blockDim.x) {
        double s = 0.0;
        for (uint64_t g = 0; g < ng; ++g) s = __dadd_rn(s, w.groups[g * width + col]);
        w.tot[col] = s;
    }
    finish_call(w.tot, w.fin);  // (its first __syncthreads publishes tot to the block)
}

}  // namespace ltg
