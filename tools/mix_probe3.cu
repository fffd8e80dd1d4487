// Which pipe do int->fp64 conversions and bfind use on sm_100 (development
// probe; see mix_probe2.cu): 4 DMUL+DADD chains per thread plus, per FP64
// pair, I independent ops of kind K on integer chains; 8 CTAs x 128 thr/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int K>
__device__ __forceinline__ void iop(uint32_t& u, uint32_t& v) {
    if (K == 0) { u ^= v; v += 0x9E3779B9u; }   // control: the ALU work of K=1,2 without the cvt
    if (K == 1) {                                // cvt.rn.f64.s64 (I2F.F64.S64)
        const long long w = ((long long)(int)u << 20) | v;
        double d; asm("cvt.rn.f64.s64 %0, %1;" : "=d"(d) : "l"(w));
        u ^= (uint32_t)__double2hiint(d); v += 0x9E3779B9u;
    }
    if (K == 2) {                                // cvt.rn.f64.u32 (I2F.F64.U32)
        double d; asm("cvt.rn.f64.u32 %0, %1;" : "=d"(d) : "r"(u));
        u ^= (uint32_t)__double2hiint(d); v += 0x9E3779B9u;
    }
    if (K == 3) {                                // bfind.u32 (FLO)
        uint32_t b; asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(u | 1u));
        u ^= b + v; v += 0x9E3779B9u;
    }
    if (K == 4) {                                // 64-bit compare + select (ISETP.EX pair)
        const long long w = ((long long)(int)u << 20) | v;
        u ^= (w > 3828157131937710LL || w < -3828157131937710LL) ? 1u : 0u; v += 0x9E3779B9u;
    }
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
    printf("%-14s x%d per fp64 pair: %.3e fp64 thread-inst/s (%.1f lanes/clk/SM)\n", name, I, rate,
           rate / (148 * 1.965e9));
}
int main() {
    double* o; cudaMalloc(&o, 8);
    run<0, 1>(o, "control"); run<0, 2>(o, "control");
    run<1, 1>(o, "cvt.f64.s64"); run<1, 2>(o, "cvt.f64.s64");
    run<2, 1>(o, "cvt.f64.u32"); run<2, 2>(o, "cvt.f64.u32");
    run<3, 1>(o, "bfind"); run<3, 2>(o, "bfind");
    run<4, 1>(o, "cmp64"); run<4, 2>(o, "cmp64");
    return 0;
}
