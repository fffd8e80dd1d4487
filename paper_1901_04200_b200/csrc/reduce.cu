// reduce.cu — deterministic reductions, finalisation, and the stand-alone
// normal generator behind ltg_fill_normals.
//
// Chunk partial tables [n_chunks][width] are reduced in a fixed order that
// depends only on the total path count: chunks are summed sequentially in
// groups of kGroup, then the group sums sequentially. Together with the fixed
// per-chunk order inside the pass kernels this makes E[y], G and ∇G bitwise
// independent of the number of GPUs, as the reference's BatchSums make them
// independent of worker_threads (expectation.hpp:105-122).
#include <cuda_runtime.h>

#include "kernels.h"
#include "rng.cuh"

namespace ltg {
namespace {

__global__ void reduce_groups_kernel(const double* __restrict__ table, uint64_t n_chunks,
                                     uint32_t width, uint64_t n_groups,
                                     double* __restrict__ groups) {
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_groups * width) return;
    const uint64_t g = idx / width;
    const uint32_t col = (uint32_t)(idx % width);
    const uint64_t c0 = g * kGroup;
    const uint64_t c1 = min(c0 + (uint64_t)kGroup, n_chunks);
    double s = 0.0;
    for (uint64_t c = c0; c < c1; ++c) s += table[c * width + col];
    groups[g * width + col] = s;
}

__global__ void reduce_final_kernel(const double* __restrict__ groups, uint64_t n_groups,
                                    uint32_t width, double* __restrict__ out) {
    const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= width) return;
    double s = 0.0;
    for (uint64_t g = 0; g < n_groups; ++g) s += groups[g * width + col];
    out[col] = s;
}

// means_from_sums (expectation.hpp:251-269) and lambda / G (:329-334)
__global__ void finalize_means_kernel(const double* __restrict__ totals, uint32_t m,
                                      uint64_t paths, const double* __restrict__ targets,
                                      double* __restrict__ res) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double P = (double)paths;
    double* means = res + 1;
    double* se = res + 1 + m;
    double* lambda = res + 1 + 2 * m;
    for (uint32_t o = 0; o < m; ++o) {
        const double mean = __ddiv_rn(totals[o], P);
        means[o] = mean;
        if (paths > 1) {
            double var = __ddiv_rn(__dsub_rn(totals[m + o], __dmul_rn(__dmul_rn(P, mean), mean)),
                                   __dsub_rn(P, 1.0));
            var = var > 0.0 ? var : 0.0;
            se[o] = __dsqrt_rn(__ddiv_rn(var, P));
        } else {
            se[o] = 0.0;
        }
    }
    double G = 0.0;
    if (targets) {
        for (uint32_t o = 0; o < m; ++o) {
            const double l = __dsub_rn(means[o], targets[o]);
            lambda[o] = l;
            G = __dadd_rn(G, __dmul_rn(__dmul_rn(0.5, l), l));
        }
    }
    res[0] = G;
}

__global__ void finalize_grad_kernel(const double* __restrict__ totals, uint32_t M,
                                     uint64_t paths, double* __restrict__ grad) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < M) grad[j] = __ddiv_rn(totals[j], (double)paths);
}

// PhiloxNormalSource::fill for a path range through the production
// generator (gen_segment), one path per thread.
constexpr int KF = 16;
__global__ void __launch_bounds__(kBlock) fill_normals_kernel(
    const RngTables* tables, RngConsts rc, uint32_t seed_lo, uint32_t seed_hi, int antithetic,
    uint64_t path0, uint64_t npaths, uint32_t dim, double* __restrict__ out) {
    __shared__ RngTables sh;
    __shared__ double zbuf[2 * KF * kBlock];
    __shared__ uint16_t wlist[kWarps * 64 * KF];
    load_tables(&sh, tables);
    __syncthreads();
    const uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    const uint64_t path = path0 + (i < npaths ? i : npaths - 1);
    const uint64_t base = antithetic ? path >> 1 : path;
    const bool neg = antithetic && (path & 1u);
    const uint32_t pairs = (dim + 1) / 2;
    double* zb = zbuf + threadIdx.x;
    uint16_t* wl = wlist + (threadIdx.x >> 5) * 64 * KF;
    for (uint32_t k0 = 0; k0 < pairs; k0 += KF) {
        const int kn = (int)min((uint32_t)KF, pairs - k0);
        gen_segment<KF>(base, neg, k0, kn, seed_lo, seed_hi, zb, wl, sh, rc);
        if (i < npaths)
            for (int s = 0; s < 2 * kn; ++s) {
                const uint32_t slot = 2 * k0 + s;
                if (slot < dim) out[i * dim + slot] = zb[s * kBlock];
            }
    }
}

// inverse_normal_cdf (rng.hpp:45-85) of given uniforms through the device
// AS241 (diagnostic: the path kernels fuse it with Philox in gen_segment).
// p must be of the generator's form (2n+1)*2^-53, so q = p - 0.5 is exact.
__global__ void inverse_normal_kernel(const RngTables* tables, RngConsts rc, const double* p,
                                      uint64_t n, double* z) {
    __shared__ RngTables sh;
    load_tables(&sh, tables);
    __syncthreads();
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double q = __dsub_rn(p[i], 0.5);
    z[i] = fabs(q) <= rc.lit_qmax ? as241_central(q, rc) : as241_tail(q, sh, rc);
}

// tangent mode: grad[d] = (sum_i lambda_i * J[i*M + d]) / P, i ascending
__global__ void finalize_grad_tangent_kernel(const double* J, const double* lambda, uint32_t m,
                                             uint32_t M, uint64_t paths, double* grad) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= M) return;
    double t = 0.0;
    for (uint32_t i = 0; i < m; ++i) t = __dadd_rn(t, __dmul_rn(lambda[i], J[(size_t)i * M + d]));
    grad[d] = __ddiv_rn(t, (double)paths);
}

}  // namespace

cudaError_t launch_reduce_chunks(const double* table, uint64_t n_chunks, uint32_t width,
                                 double* group_scratch, double* out, cudaStream_t s) {
    const uint64_t n_groups = (n_chunks + kGroup - 1) / kGroup;
    const uint64_t n = n_groups * width;
    reduce_groups_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(table, n_chunks, width,
                                                                      n_groups, group_scratch);
    reduce_final_kernel<<<(width + 127) / 128, 128, 0, s>>>(group_scratch, n_groups, width, out);
    return cudaGetLastError();
}

cudaError_t launch_finalize_means(const double* totals, uint32_t m, uint64_t paths,
                                  const double* targets, double* res, cudaStream_t s) {
    finalize_means_kernel<<<1, 32, 0, s>>>(totals, m, paths, targets, res);
    return cudaGetLastError();
}

cudaError_t launch_finalize_grad(const double* totals, uint32_t M, uint64_t paths, double* grad,
                                 cudaStream_t s) {
    finalize_grad_kernel<<<(M + 127) / 128, 128, 0, s>>>(totals, M, paths, grad);
    return cudaGetLastError();
}

cudaError_t launch_fill_normals(const RngTables* tables, const RngConsts& rc, uint32_t seed_lo,
                                uint32_t seed_hi, int antithetic, uint64_t path0, uint64_t npaths,
                                uint32_t dim, double* out, cudaStream_t s) {
    if (npaths == 0 || dim == 0) return cudaSuccess;
    fill_normals_kernel<<<(unsigned)((npaths + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        tables, rc, seed_lo, seed_hi, antithetic, path0, npaths, dim, out);
    return cudaGetLastError();
}

cudaError_t launch_inverse_normal(const RngTables* tables, const RngConsts& rc, const double* p,
                                   uint64_t n, double* z, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    inverse_normal_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(tables, rc, p, n, z);
    return cudaGetLastError();
}

cudaError_t launch_finalize_grad_tangent(const double* J, const double* lambda, uint32_t m,
                                         uint32_t M, uint64_t paths, double* grad,
                                         cudaStream_t s) {
    finalize_grad_tangent_kernel<<<(M + 127) / 128, 128, 0, s>>>(J, lambda, m, M, paths, grad);
    return cudaGetLastError();
}

}  // namespace ltg
