// Checks rng.cuh's ddiv_fast / dsqrt_ref / dsqrt_fast against CUDA's IEEE
// __ddiv_rn / __dsqrt_rn on random operands (development probe).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1901_04200_b200/csrc/rng.cuh"
using namespace ltg;
__device__ unsigned long long xs(unsigned long long& s) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
__global__ void k(unsigned long long* bad, int iters) {
    unsigned long long s = 0x9E3779B97F4A7C15ULL ^ (blockIdx.x * 1315423911ull + threadIdx.x);
    unsigned long long nb[3] = {0, 0, 0};
    for (int i = 0; i < iters; ++i) {
        const double u = (double)(xs(s) >> 11) * 0x1p-53;
        const double v = (double)(xs(s) >> 11) * 0x1p-53;
        // AS241-like ranges: numerator 1e-16 .. 1e4, denominator 1 .. 1e6
        const double a = ldexp(1.0 + u, (int)(xs(s) % 70) - 55) * ((xs(s) & 1) ? -1.0 : 1.0);
        const double b = ldexp(1.0 + v, (int)(xs(s) % 20));
        if (__double_as_longlong(ddiv_fast(a, b)) != __double_as_longlong(__ddiv_rn(a, b))) ++nb[0];
        // sqrt over the whole positive range incl. 0 and denormals
        const int e = (int)(xs(s) % 2100) - 1075;
        double x = ldexp(1.0 + u, e);
        if ((xs(s) & 255) == 0) x = 0.0;
        if (__double_as_longlong(dsqrt_ref(x)) != __double_as_longlong(__dsqrt_rn(x))) ++nb[1];
        const double t = 2.5 + 35.0 * v;  // AS241 tail range
        if (__double_as_longlong(dsqrt_fast(t)) != __double_as_longlong(__dsqrt_rn(t))) ++nb[2];
    }
    for (int j = 0; j < 3; ++j) if (nb[j]) atomicAdd(&bad[j], nb[j]);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    k<<<blocks, threads>>>(d, iters);
    unsigned long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("{\"samples\": %llu, \"ddiv_mismatch\": %llu, \"dsqrt_ref_mismatch\": %llu, \"dsqrt_fast_mismatch\": %llu, \"err\": \"%s\"}\n",
           (unsigned long long)blocks * threads * iters, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
