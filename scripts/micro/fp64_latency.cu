// Microbenchmark: FP64 latencies and throughputs on the device (one warp / full SM).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dfma(double* out, long long* cyc, int n, double a, double b)
{
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_dadd(double* out, long long* cyc, int n, double a)
{
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) x = x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_rcp(double* out, long long* cyc, int n)
{
    double x = 1.0 + threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP>
__global__ void tput_dfma(double* out, long long* cyc, int n, double a, double b)
{
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMallocManaged(&cyc, 64);
    const int n = 4096;
    chain_dfma<<<1, 32>>>(out, cyc, n, 0.999, 1e-9);
    cudaDeviceSynchronize();
    chain_dfma<<<1, 32>>>(out, cyc, n, 0.999, 1e-9);
    cudaDeviceSynchronize();
    printf("DFMA dependent latency: %.2f cycles\n", (double)cyc[0] / n);
    chain_dadd<<<1, 32>>>(out, cyc, n, 1e-9);
    cudaDeviceSynchronize();
    printf("DADD dependent latency: %.2f cycles\n", (double)cyc[0] / n);
    chain_rcp<<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
    printf("MUFU.RCP64H dependent latency: %.2f cycles\n", (double)cyc[0] / n);
    // one warp per SMSP (4 warps / CTA), ILP sweep: cycles per DFMA per warp
    tput_dfma<1><<<1, 128>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("1 warp/SMSP ILP1: %.2f cyc per warp-DFMA\n", (double)cyc[0] / n / 1);
    tput_dfma<2><<<1, 128>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("1 warp/SMSP ILP2: %.2f cyc per warp-DFMA\n", (double)cyc[0] / n / 2);
    tput_dfma<4><<<1, 128>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("1 warp/SMSP ILP4: %.2f cyc per warp-DFMA\n", (double)cyc[0] / n / 4);
    tput_dfma<8><<<1, 128>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("1 warp/SMSP ILP8: %.2f cyc per warp-DFMA\n", (double)cyc[0] / n / 8);
    tput_dfma<4><<<1, 512>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("4 warps/SMSP ILP4: %.2f cyc per 4 warp-DFMA (per SMSP)\n", (double)cyc[0] / n / 4);
    tput_dfma<2><<<1, 1024>>>(out, cyc, n, 0.999, 1e-9); cudaDeviceSynchronize();
    printf("8 warps/SMSP ILP2: %.2f cyc per 8 warp-DFMA (per SMSP)\n", (double)cyc[0] / n / 2);
    return 0;
}
