// Dependent-chain latency (cycles) of FP64 ops on this GPU (development probe).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, double a, double b, int n, int which) {
    double x = threadIdx.x * 1e-9 + 1.0, y = 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (which == 0) x = __fma_rn(x, a, b);
        else if (which == 1) x = __dadd_rn(x, b);
        else if (which == 2) x = __dmul_rn(x, a);
        else if (which == 3) x = __ddiv_rn(b, x);
        else if (which == 4) x = __dsqrt_rn(x);
        else if (which == 5) x = __dmul_rn(__dadd_rn(x, b), a);
        else if (which == 6) { x = rsqrt(x); }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"dfma", "dadd", "dmul", "ddiv_rn", "dsqrt_rn", "dadd+dmul", "rsqrt"};
    for (int w = 0; w < 7; ++w) {
        int n = 4096; long long cyc = 0;
        chain<<<1, 32>>>(o, c, 0.9999999, 1e-9, n, w);
        chain<<<1, 32>>>(o, c, 0.9999999, 1e-9, n, w);
        cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
        printf("%-10s %.2f cycles/op (1 warp, dependent)\n", names[w], (double)cyc / n);
    }
    // throughput with 1 warp, 8 independent chains
    return 0;
}
