// Which integer instructions compete with FP64 on sm_100 (development probe):
// 4 independent DMUL+DADD chains per thread plus, per FP64 pair, one
// independent integer op of kind K on its own chain; 8 CTAs x 128 threads/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int K>
__device__ __forceinline__ void iop(uint32_t& u, uint32_t& v) {
    if (K == 0) { uint64_t p; asm("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p) : "r"(u)); u = (uint32_t)p ^ v; v = (uint32_t)(p >> 32); }
    if (K == 1) asm("mul.hi.u32 %0, %0, 0xD2511F53;" : "+r"(u));
    if (K == 2) asm("mul.lo.u32 %0, %0, 0xD2511F53;" : "+r"(u));
    if (K == 3) asm("xor.b32 %0, %0, %1;" : "+r"(u) : "r"(v));
    if (K == 4) asm("add.u32 %0, %0, %1;" : "+r"(u) : "r"(v));
    if (K == 5) asm("lop3.b32 %0, %0, %1, 0x5bd1e995, 0x96;" : "+r"(u) : "r"(v));
    if (K == 6) asm("mad.lo.u32 %0, %0, 0xD2511F53, %1;" : "+r"(u) : "r"(v));
    if (K == 7) { float f = __uint_as_float(u); asm("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f)); u = __float_as_uint(f); }
}
template <int K, int I>
__global__ void __launch_bounds__(128) k(double* out, int iters, double a, double b) {
    constexpr int C = 4;
    double x[C];
    uint32_t u[C], v[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { x[i] = threadIdx.x * 1e-3 + i; u[i] = threadIdx.x * 2654435761u + i; v[i] = blockIdx.x + 3 * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) {
            x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
#pragma unroll
            for (int j = 0; j < I; ++j) iop<K>(u[i], v[i]);
        }
    }
    double s = 0; uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) { s += x[i]; t ^= u[i] ^ v[i]; }
    if (s == 12345.678 || t == 7) out[0] = s + t;
}
template <int K, int I>
void run(double* o, const char* name) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = 148 * 8, iters = 4096;
    k<K, I><<<grid, 128>>>(o, 64, 0.9999999, 1e-9);
    cudaEventRecord(e0); k<K, I><<<grid, 128>>>(o, iters, 0.9999999, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double rate = double(grid) * 128 * iters * 4 * 2 / (ms * 1e-3);
    printf("%-12s x%d per fp64 pair: %.3e fp64 thread-inst/s (%.1f lanes/clk/SM)\n", name, I, rate,
           rate / (148 * 1.965e9));
}
int main() {
    double* o; cudaMalloc(&o, 8);
    run<4, 0>(o, "none");
    run<0, 1>(o, "mul.wide"); run<0, 2>(o, "mul.wide");
    run<1, 1>(o, "mul.hi"); run<1, 2>(o, "mul.hi");
    run<2, 1>(o, "mul.lo"); run<2, 2>(o, "mul.lo");
    run<6, 1>(o, "mad.lo"); run<6, 2>(o, "mad.lo");
    run<3, 2>(o, "xor"); run<3, 4>(o, "xor");
    run<5, 2>(o, "lop3"); run<5, 4>(o, "lop3");
    run<4, 2>(o, "add"); run<4, 4>(o, "add");
    run<7, 2>(o, "ffma"); run<7, 4>(o, "ffma");
    return 0;
}
