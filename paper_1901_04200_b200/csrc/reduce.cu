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
#include "finish.cuh"
#include "rng.cuh"

namespace ltg {
namespace {

// Column sums of rows [r0, r1) of a row-major [*][width] table, each in
// ascending row order (the fixed order the results depend on). The CTA
// stages a kTileRows x tw tile through shared memory with independent,
// coalesced loads, then thread t adds column t of the tile in row order, so a
// column costs one memory latency per tile instead of one per row.
constexpr int kTileRows = 64, kTileCols = 64;
__device__ void ordered_column_sums(const double* table, uint64_t r0, uint64_t r1,
                                    uint32_t width, double* out,
                                    double (*tile)[kTileCols]) {
    for (uint32_t c0 = 0; c0 < width; c0 += kTileCols) {
        const uint32_t tw = min((uint32_t)kTileCols, width - c0);
        double s = 0.0;
        for (uint64_t rb = r0; rb < r1; rb += kTileRows) {
            const uint32_t tr = (uint32_t)min((uint64_t)kTileRows, r1 - rb);
            for (uint32_t e = threadIdx.x; e < tr * tw; e += blockDim.x) {
                const uint32_t r = e / tw, c = e - r * tw;
                tile[r][c] = table[(rb + r) * width + c0 + c];
            }
            __syncthreads();
            if (threadIdx.x < tw)
                for (uint32_t r = 0; r < tr; ++r) s = __dadd_rn(s, tile[r][threadIdx.x]);
            __syncthreads();
        }
        if (threadIdx.x < tw) out[c0 + threadIdx.x] = s;
    }
}

// one CTA per group of kGroup chunk rows
__global__ void __launch_bounds__(kFinishThreads) reduce_groups_kernel(
    const double* __restrict__ table, uint64_t n_chunks, uint32_t width,
    double* __restrict__ groups) {
    __shared__ double tile[kTileRows][kTileCols];
    const uint64_t g = blockIdx.x;
    const uint64_t c0 = g * kGroup;
    const uint64_t c1 = min(c0 + (uint64_t)kGroup, n_chunks);
    ordered_column_sums(table, c0, c1, width, groups + g * width, tile);
}

__global__ void __launch_bounds__(kFinishThreads) reduce_final_kernel(
    const double* __restrict__ groups, uint64_t n_groups, uint32_t width, double* out, Finish f) {
    __shared__ double tile[kTileRows][kTileCols];
    ordered_column_sums(groups, 0, n_groups, width, out, tile);
    finish_call(out, f);
}


// PhiloxNormalSource::fill for a path range through the production
// generator (gen_segment), one path per thread.
constexpr int KF = 16;
__global__ void __launch_bounds__(kBlock) fill_normals_kernel(
    const RngTables* tables, RngConsts rc, PhiloxKeys rk, int antithetic,
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
        gen_segment<KF>(base, neg, k0, kn, rk, zb, wl, sh, rc);
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

}  // namespace

cudaError_t launch_reduce_chunks(const double* table, uint64_t n_chunks, uint32_t width,
                                 double* group_scratch, double* out, const Finish& fin,
                                 cudaStream_t s) {
    const uint64_t n_groups = (n_chunks + kGroup - 1) / kGroup;
    const cudaError_t e = launch_kernel(reduce_groups_kernel, (unsigned)n_groups, kFinishThreads,
                                        0, s, table, n_chunks, width, group_scratch);
    if (e != cudaSuccess) return e;
    return launch_kernel(reduce_final_kernel, 1, kFinishThreads, 0, s, (const double*)group_scratch,
                         n_groups, width, out, fin);
}

cudaError_t launch_fill_normals(const RngTables* tables, const RngConsts& rc, uint32_t seed_lo,
                                uint32_t seed_hi, int antithetic, uint64_t path0, uint64_t npaths,
                                uint32_t dim, double* out, cudaStream_t s) {
    if (npaths == 0 || dim == 0) return cudaSuccess;
    fill_normals_kernel<<<(unsigned)((npaths + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        tables, rc, make_philox_keys(seed_lo, seed_hi), antithetic, path0, npaths, dim, out);
    return cudaGetLastError();
}

cudaError_t launch_inverse_normal(const RngTables* tables, const RngConsts& rc, const double* p,
                                   uint64_t n, double* z, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    inverse_normal_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(tables, rc, p, n, z);
    return cudaGetLastError();
}

}  // namespace ltg
