// fdg_probe.cu -- sustained FP64 FMA throughput of the device.
//
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks but no FP64 figure;
// the roofline of the volume integral needs one.  This is a
// DFMA-only loop: 8 independent chains per thread (enough ILP to cover the
// pipe latency), 2 flop per DFMA, timed with CUDA events on the given stream.
#include <cuda_runtime.h>

#include "../../include/fdg.h"

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double s)
{
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double c = 0.999999;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, c, s); a1 = fma(a1, c, s); a2 = fma(a2, c, s); a3 = fma(a3, c, s);
        a4 = fma(a4, c, s); a5 = fma(a5, c, s); a6 = fma(a6, c, s); a7 = fma(a7, c, s);
    }
    double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 123.456) out[0] = r;  // keep the loop alive
}

extern "C" int fdg_fp64_probe(double* tflops, void* stream)
{
    if (!tflops) return FDG_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return FDG_ERR_CUDA;
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    dfma_loop<<<blocks, threads, 0, s>>>(out, iters, 1e-12);  // warm-up (clocks ramp)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, s);
        dfma_loop<<<blocks, threads, 0, s>>>(out, iters, 1e-12);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return FDG_ERR_CUDA;
    const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    return FDG_OK;
}
