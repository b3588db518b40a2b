// DFMA throughput microbenchmark (B200 fp64 CUDA-core peak, the roofline denominator for the
// FFT-bound kernels). 8 independent FMA chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1 << 16, blocks = sms * 8, threads = 256;
    k<<<blocks, threads>>>(d, 100, 0.999, 0.001);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
    return 0;
}
