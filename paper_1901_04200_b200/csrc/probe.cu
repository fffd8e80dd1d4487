// probe.cu — measured FP64 issue rate of this GPU (the roofline denominator
// for the FP64-bound ∇G kernels; MEASURED_PEAKS.json has no FP64 entry).
// Each thread runs 8 independent DFMA chains; rate = thread-DFMAs / second.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lanetape_b200.h"

namespace {

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" int ltg_probe_fp64_rate(int device, double* dfma_per_s, double* sm_clock_hz) {
    if (cudaSetDevice(device) != cudaSuccess) return LTG_ECUDA;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dfma_kernel, 256, 0);
    double* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return LTG_ECUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * (per_sm > 0 ? per_sm : 1);
    const int iters = 1 << 14;
    dfma_kernel<<<grid, 256>>>(out, 256, 0.999999, 1e-7);  // warm-up / clock ramp
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return LTG_ECUDA;
    *dfma_per_s = double(grid) * 256.0 * iters * 8.0 / (best * 1e-3);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
    if (sm_clock_hz) *sm_clock_hz = khz * 1e3;
    return LTG_OK;
}
