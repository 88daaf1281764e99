// fp64_peak.cu -- FP64 FMA throughput microbenchmark (the "alu" peak of DESIGN.md).
// Each thread runs 8 independent DFMA chains; grid = 148 SMs x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters, double a, double b)
{
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
    if (s == 123.456) out[0] = s;
}
int main()
{
    double *d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, thr = 256, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, thr>>>(d, 100, 0.999, 1e-3);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<<<blocks, thr>>>(d, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * (double)iters * blocks * thr;
    printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d}\n", flops / best / 1e9, best, sms);
    return 0;
}
