// Does the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) run alongside DFMA?
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, double s) {
    double a = s + threadIdx.x * 1e-9, b = 0.5;
    double d[8][2] = {};
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += d[k][0] + d[k][1];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_dfma(double *out, double s) {
    double a[8]; const double b = 0.999999999, c = 1e-10;
    for (int k = 0; k < 8; ++k) a[k] = s + k + threadIdx.x * 1e-9;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { a[k] = fma(a[k], b, c); a[k] = fma(a[k], b, c); }
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
// both in one kernel: per iteration 8 DMMA + 16 DFMA
__global__ void k_both(double *out, double s) {
    double x = s + threadIdx.x * 1e-9, y = 0.5;
    double d[8][2] = {};
    double a[8]; const double b = 0.999999999, c = 1e-10;
    for (int k = 0; k < 8; ++k) a[k] = s + k + threadIdx.x * 1e-9;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            dmma(d[k][0], d[k][1], x, y);
            a[k] = fma(a[k], b, c); a[k] = fma(a[k], b, c);
        }
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += d[k][0] + d[k][1] + a[k];
    if (r == 1.2345) out[0] = r;
}

template <typename K>
float run(K k) {
    double *o; cudaMalloc(&o, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms * 8, 256>>>(o, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<<<sms * 8, 256>>>(o, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); cudaFree(o);
    printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return ms;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double warps = sms * 8 * 8.0, thr = sms * 8 * 256.0;
    float t1 = run(k_dmma), t2 = run(k_dfma), t3 = run(k_both);
    double dmma_flops = warps * ITERS * 8 * 512.0, dfma_flops = thr * ITERS * 16 * 2.0;
    printf("dmma only: %.2f TFLOP/s (%.3f ms)\n", dmma_flops / t1 / 1e9, t1);
    printf("dfma only: %.2f TFLOP/s (%.3f ms)\n", dfma_flops / t2 / 1e9, t2);
    printf("both: %.3f ms; sum-of-separate %.3f ms; combined %.2f TFLOP/s\n", t3, t1 + t2,
           (dmma_flops + dfma_flops) / t3 / 1e9);
}
