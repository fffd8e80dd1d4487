// Latency of the pieces of a small call replayed from a CUDA graph
// (development probe): a chain of K short kernels with and without the
// call's H2D copy, flag memset and D2H copy, synchronised by
// cudaStreamSynchronize or by spinning on a word the last kernel writes to
// mapped pinned memory. Prints the mean wall time per call of each form.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/graph_probe tools/graph_probe.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__global__ void work(double* buf, int iters, volatile unsigned* done, unsigned seq) {
    double v = buf[threadIdx.x];
    for (int i = 0; i < iters; ++i) v = v * 0.999 + 1e-3;
    buf[threadIdx.x] = v;
    if (done && threadIdx.x == 0 && blockIdx.x == 0) {
        __threadfence_system();
        *done = seq;
    }
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double *d, *dx, *hst;
    unsigned* dflags;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&dx, 4096);
    cudaMalloc(&dflags, 256);
    cudaHostAlloc(&hst, 8192, cudaHostAllocMapped);
    unsigned* hdone;
    cudaHostAlloc(&hdone, 64, cudaHostAllocMapped);
    unsigned* ddone;
    cudaHostGetDevicePointer(&ddone, hdone, 0);
    const int K = 6, iters = 20;
    for (int form = 0; form < 8; ++form) {
        // form bit 0: H2D + memset + D2H nodes; bit 1: spin on the mapped word; bit 2: 2 kernels
        const bool copies = form & 1, spin = form & 2;
        const int nk = (form & 4) ? 2 : K;
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        if (copies) {
            cudaMemcpyAsync(dx, hst, 200, cudaMemcpyHostToDevice, s);
            cudaMemsetAsync(dflags, 0, 64, s);
        }
        for (int k = 0; k < nk; ++k)
            work<<<148, 128, 0, s>>>(d, iters, (spin && k == nk - 1) ? ddone : nullptr, 1);
        if (copies) cudaMemcpyAsync(hst + 512, d, 600, cudaMemcpyDeviceToHost, s);
        cudaStreamEndCapture(s, &g);
        cudaGraphExec_t ge;
        cudaGraphInstantiate(&ge, g, 0);
        for (int w = 0; w < 50; ++w) {
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
        }
        const int N = 2000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        double dev = 0;
        auto t0 = std::chrono::high_resolution_clock::now();
        for (int i = 0; i < N; ++i) {
            if (spin) {
                *(volatile unsigned*)hdone = 0;
                cudaGraphLaunch(ge, s);
                while (*(volatile unsigned*)hdone == 0) {
                }
            } else {
                cudaGraphLaunch(ge, s);
                cudaStreamSynchronize(s);
            }
        }
        auto t1 = std::chrono::high_resolution_clock::now();
        cudaStreamSynchronize(s);
        // device span of the kernels alone
        cudaEventRecord(e0, s);
        for (int k = 0; k < nk; ++k) work<<<148, 128, 0, s>>>(d, iters, nullptr, 1);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        dev = ms * 1e3;
        printf("form %d (kernels %d, copies %d, spin %d): wall %.2f us/call; eager kernel span %.2f us\n",
               form, nk, (int)copies, (int)spin,
               std::chrono::duration<double, std::micro>(t1 - t0).count() / N, dev);
    }
    return 0;
}
