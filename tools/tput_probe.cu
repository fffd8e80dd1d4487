// FP64 issue throughput by instruction kind (development probe): 8 independent
// chains per thread, 148*8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void __launch_bounds__(256) k(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (W == 0) x[i] = __fma_rn(x[i], a, b);
            if (W == 1) x[i] = __dadd_rn(x[i], b);
            if (W == 2) x[i] = __dmul_rn(x[i], a);
            if (W == 3) x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
template <int W>
double run(double* o, const char* name, int per_iter) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = 148 * 8, iters = 8192;
    k<W><<<grid, 256>>>(o, 64, 0.9999999, 1e-9);
    cudaEventRecord(e0); k<W><<<grid, 256>>>(o, iters, 0.9999999, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double rate = double(grid) * 256 * iters * 8 * per_iter / (ms * 1e-3);
    printf("%-10s %.3e thread-inst/s  (%.1f lanes/clk/SM at 1965 MHz)\n", name, rate, rate / (148 * 1.965e9));
    return rate;
}
int main() {
    double* o; cudaMalloc(&o, 8);
    run<0>(o, "dfma", 1); run<1>(o, "dadd", 1); run<2>(o, "dmul", 1); run<3>(o, "dmul+dadd", 2);
    return 0;
}
