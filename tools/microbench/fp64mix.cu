// DMUL vs DFMA throughput on B200 (8 independent chains per thread, 8 warps per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>  // 0 DFMA, 1 DMUL, 2 mixed 3 DFMA : 1 DMUL, 3 DMUL written as DFMA with -0.0 addend
__global__ void k(double *out, int n) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = out[i] + threadIdx.x;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) a[i] = fma(a[i], b, c);
            else if (KIND == 1) a[i] = a[i] * b;
            else if (KIND == 2) a[i] = (i % 4 == 3) ? a[i] * b : fma(a[i], b, c);
            else a[i] = fma(a[i], b, -0.0);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1234.5) out[threadIdx.x] = s;
}
int main() {
    double *d; cudaMalloc(&d, 1 << 16); cudaMemset(d, 0, 1 << 16);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 20000;
    const char *names[4] = {"DFMA", "DMUL", "3DFMA:1DMUL", "DMUL-as-DFMA"};
    for (int kind = 0; kind < 4; ++kind)
        for (int wps : {8, 16}) {
            float ms;
            auto run = [&]() {
                if (kind == 0) k<0><<<nsm, 32 * wps>>>(d, n);
                if (kind == 1) k<1><<<nsm, 32 * wps>>>(d, n);
                if (kind == 2) k<2><<<nsm, 32 * wps>>>(d, n);
                if (kind == 3) k<3><<<nsm, 32 * wps>>>(d, n);
            };
            run();
            cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)nsm * 32 * wps * n * 8;
            printf("%-14s warps/SM=%2d: %.2f T instr/s\n", names[kind], wps, ops / ms / 1e9);
        }
    return 0;
}
