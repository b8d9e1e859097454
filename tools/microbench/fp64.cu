// FP64 pipe microbenchmarks on B200 (sm_100a): DFMA latency / throughput, DMMA (mma.sync
// m8n8k4 f64) throughput, and DFMA + DMMA issued concurrently by different warps.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double *out, int n, long long *cyc) {
    double a = out[0], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) a = fma(a, b, c);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x + 1] = a;
}

template <int ILP>
__global__ void tput_dfma(double *out, int n) {
    double a[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) a[k] = out[k] + threadIdx.x;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += a[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void tput_dmma(double *out, int n) {
    double a = out[0] + threadIdx.x, b = 1.0000001;
    double c[4][2] = {};
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[threadIdx.x] = s;
}

// even warps DFMA, odd warps DMMA
__global__ void mixed(double *out, int n, int nm) {
    const int w = threadIdx.x >> 5;
    if (w & 1) {
        double a = out[0] + threadIdx.x, b = 1.0000001;
        double c[4][2] = {};
        for (int i = 0; i < nm; ++i) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
        double s = 0;
        for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
        if (s == 12345.0) out[threadIdx.x] = s;
    } else {
        double a[8];
        for (int k = 0; k < 8; ++k) a[k] = out[k] + threadIdx.x;
        const double b = 1.0000001, c = 1e-9;
        for (int i = 0; i < n; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
        double s = 0;
        for (int k = 0; k < 8; ++k) s += a[k];
        if (s == 12345.0) out[threadIdx.x] = s;
    }
}

int main() {
    double *d;
    long long *cyc;
    cudaMalloc(&d, 1 << 20);
    cudaMemset(d, 0, 1 << 20);
    cudaMalloc(&cyc, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // latency
    lat_dfma<<<1, 32>>>(d, 1000, cyc);
    lat_dfma<<<1, 32>>>(d, 10000, cyc);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)c / (10000 * 16));
    // throughput sweep
    const int n = 20000;
    for (int wps : {4, 8, 12, 16, 32}) {
        tput_dfma<8><<<nsm, 32 * wps>>>(d, 100);
        cudaEventRecord(e0);
        tput_dfma<8><<<nsm, 32 * wps>>>(d, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * nsm * 32.0 * wps * n * 8;
        printf("DFMA ILP8 warps/SM=%2d: %.2f TFLOP/s\n", wps, flops / ms / 1e9);
    }
    for (int wps : {4, 8, 12}) {
        tput_dfma<2><<<nsm, 32 * wps>>>(d, 100);
        cudaEventRecord(e0);
        tput_dfma<2><<<nsm, 32 * wps>>>(d, n * 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * nsm * 32.0 * wps * n * 4 * 2;
        printf("DFMA ILP2 warps/SM=%2d: %.2f TFLOP/s\n", wps, flops / ms / 1e9);
    }
    for (int wps : {4, 8, 16}) {
        tput_dmma<<<nsm, 32 * wps>>>(d, 100);
        cudaEventRecord(e0);
        tput_dmma<<<nsm, 32 * wps>>>(d, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 4 * (double)n * nsm * wps;
        printf("DMMA m8n8k4 warps/SM=%2d: %.2f TFLOP/s\n", wps, flops / ms / 1e9);
    }
    // mixed: 8 DFMA warps + 8 DMMA warps per SM; compare time with each alone
    {
        const int nm = n / 2;
        mixed<<<nsm, 512>>>(d, 100, 50);
        cudaEventRecord(e0);
        mixed<<<nsm, 512>>>(d, n, nm);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double f1 = 2.0 * nsm * 32.0 * 8 * n * 8, f2 = 2.0 * 8 * 8 * 4 * 4 * (double)nm * nsm * 8;
        printf("mixed 8 DFMA + 8 DMMA warps: %.3f ms, DFMA %.2f + DMMA %.2f TFLOP/s\n", ms, f1 / ms / 1e9, f2 / ms / 1e9);
        mixed<<<nsm, 512>>>(d, n, 0);
        cudaEventRecord(e0);
        mixed<<<nsm, 512>>>(d, n, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  DFMA part alone: %.3f ms\n", ms);
        cudaEventRecord(e0);
        mixed<<<nsm, 512>>>(d, 0, nm);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  DMMA part alone: %.3f ms\n", ms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
