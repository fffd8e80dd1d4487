// probe.cu — measured FP64 issue rate of this GPU (the roofline denominator
// for the FP64-bound ∇G kernels; MEASURED_PEAKS.json has no FP64 entry).
// Each thread runs 8 independent chains; three instruction mixes are timed
// (DFMA; DMUL+DADD, the mix of the AS241 Horner evaluations; DADD) and the
// fastest is reported: thread-level FP64 instructions per second. The FP32
// twin (FFMA streams) is the denominator of the fp32 mode's roofline.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lanetape_b200.h"

namespace {

__global__ void __launch_bounds__(256) fp32_kernel(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;
}

template <int W>
__global__ void __launch_bounds__(256) fp64_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (W == 0) x[i] = __fma_rn(x[i], a, b);
            if (W == 1) x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
            if (W == 2) x[i] = __dadd_rn(x[i], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int W>
double rate(double* out, int grid) {
    const int iters = 1 << 13;
    const double per = W == 1 ? 2.0 : 1.0;  // FP64 instructions per chain step
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp64_kernel<W><<<grid, 256>>>(out, 256, 0.999999, 1e-7);  // warm-up / clock ramp
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        fp64_kernel<W><<<grid, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return double(grid) * 256.0 * iters * 8.0 * per / (best * 1e-3);
}

}  // namespace

extern "C" int ltg_probe_fp64_rate(int device, double* fp64_per_s, double* sm_clock_hz) {
    if (cudaSetDevice(device) != cudaSuccess) return LTG_ECUDA;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp64_kernel<0>, 256, 0);
    double* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return LTG_ECUDA;
    const int grid = sms * (per_sm > 0 ? per_sm : 1);
    double best = rate<0>(out, grid);
    const double r1 = rate<1>(out, grid), r2 = rate<2>(out, grid);
    if (r1 > best) best = r1;
    if (r2 > best) best = r2;
    const cudaError_t err = cudaGetLastError();
    cudaFree(out);
    if (err != cudaSuccess) return LTG_ECUDA;
    *fp64_per_s = best;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
    if (sm_clock_hz) *sm_clock_hz = khz * 1e3;
    return LTG_OK;
}

extern "C" int ltg_probe_fp32_rate(int device, double* fp32_per_s) {
    if (cudaSetDevice(device) != cudaSuccess) return LTG_ECUDA;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp32_kernel, 256, 0);
    float* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return LTG_ECUDA;
    const int grid = sms * (per_sm > 0 ? per_sm : 1), iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp32_kernel<<<grid, 256>>>(out, 256, 0.999999f, 1e-7f);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        fp32_kernel<<<grid, 256>>>(out, iters, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const cudaError_t err = cudaGetLastError();
    cudaFree(out);
    if (err != cudaSuccess) return LTG_ECUDA;
    *fp32_per_s = double(grid) * 256.0 * iters * 8.0 / (best * 1e-3);
    return LTG_OK;
}
