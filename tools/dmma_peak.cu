// dmma_peak.cu -- FP64 tensor-core (mma.sync m8n8k4 f64, "DMMA") throughput on sm_100a, alone
// and issued together with independent DFMA chains in the same warps: does the FP64 tensor path
// add to the FP64 FMA pipe (a design input for the sum-factorised contractions)?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both
__global__ void k(double *out, int iters, double a, double b)
{
    double c[4][2], x[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(c[i], a, b);
        }
        if (MODE != 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
}

template <int MODE>
float run(double *d, int blocks, int thr, int iters)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<blocks, thr>>>(d, 100, 0.999, 1e-3);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<MODE><<<blocks, thr>>>(d, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main()
{
    double *d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, thr = 256, iters = 20000;
    const double warps = (double)blocks * thr / 32;
    const float t0 = run<0>(d, blocks, thr, iters), t1 = run<1>(d, blocks, thr, iters), t2 = run<2>(d, blocks, thr, iters);
    const double f_mma = 2.0 * 256 * 4 * (double)iters * warps;   // 8x8x4 FMAs per mma, 4 per iteration
    const double f_fma = 2.0 * 8 * (double)iters * blocks * thr;
    printf("{\"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"both_tflops\": %.3f, \"both_ms\": %.3f, "
           "\"dmma_ms\": %.3f, \"dfma_ms\": %.3f}\n",
           f_mma / t0 / 1e9, f_fma / t1 / 1e9, (f_mma + f_fma) / t2 / 1e9, t2, t0, t1);
    return 0;
}
