// FP64 pipe microbenchmarks: operand-pattern sensitivity of DFMA/DMUL issue.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
// A: 3 distinct register operands per DFMA, 8 independent chains
__global__ void kA(double *out, double s) {
    double x[8], y[8], a[8];
    const double *in = out + 16 + (threadIdx.x & 7) * 24;
    for (int k = 0; k < 8; ++k) { x[k] = in[k]; y[k] = in[8 + k]; a[k] = in[16 + k]; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(x[k], y[k], a[k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(y[k], x[k], a[k]);
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
// B: shared constant operands (reuse-friendly)
__global__ void kB(double *out, double s) {
    double a[8]; const double b = 0.999999999, c = 1e-10;
    for (int k = 0; k < 8; ++k) a[k] = s + k + threadIdx.x * 1e-9;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
// C: DMUL with 2 distinct operands
__global__ void kC(double *out, double s) {
    double x[8], a[8];
    const double *in = out + 16 + (threadIdx.x & 7) * 24;
    for (int k = 0; k < 8; ++k) { x[k] = in[k]; a[k] = in[16 + k]; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * x[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * x[(k + 1) & 7];
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
// D: 16 chains (more ILP) with distinct operands
__global__ void kD(double *out, double s) {
    double x[16], a[16];
    const double *in = out + 16 + (threadIdx.x & 7) * 24;
    for (int k = 0; k < 16; ++k) { x[k] = in[k]; a[k] = in[8 + k]; }
    const double y = 0.9999;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fma(x[k], a[(k + 5) & 15], a[k]);
    }
    double r = 0; for (int k = 0; k < 16; ++k) r += a[k];
    if (r == 1.2345) out[0] = r * y;
}
// E: MUFU.RSQ64H throughput alongside DFMA
__global__ void kE(double *out, double s) {
    double a[8]; const double b = 0.999999999, c = 1e-10;
    double z = s + threadIdx.x * 1e-9 + 1.0;
    for (int k = 0; k < 8; ++k) a[k] = s + k + threadIdx.x * 1e-9;
    for (int i = 0; i < ITERS; ++i) {
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
        z = z + r * 1e-30;
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double r = z; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}

template <typename K>
void run(const char *name, K k, double fma_per_iter) {
    double *o; cudaMalloc(&o, 8 * 4096);
    double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 0.5 + 1e-4 * (i % 97);
    cudaMemcpy(o, h, sizeof h, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    dim3 g(sms * 8), b(256);
    k<<<g, b>>>(o, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<g, b>>>(o, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)g.x * b.x * ITERS * fma_per_iter;
    printf("%s: %.2f Gop/s (x2 = %.2f TFLOP/s)  %s\n", name, ops / ms / 1e6, 2 * ops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(o);
}

int main() {
    run("A dfma 3-distinct", kA, 16);
    run("B dfma shared    ", kB, 16);
    run("C dmul 2-distinct", kC, 16);
    run("D dfma 16 chains ", kD, 16);
    run("E rsq64h+8 dfma  ", kE, 8);
    return 0;
}
