// Are uniform-register (ULDC from __constant__) operands free of the FP64
// register-bank limit?  Each DFMA: x_k (vector) * s (per-iteration value) + acc_k.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
__constant__ double cs[8 * ITERS];

__global__ void kU(double *out) {  // s from constant memory (uniform index)
    double x[8], a[8];
    const double *in = out + 64 + (threadIdx.x & 7) * 16;
    for (int k = 0; k < 8; ++k) { x[k] = in[k]; a[k] = in[8 + k]; }
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(x[k], cs[8 * i + k], a[k]);
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
__global__ void kS(double *out) {  // s from shared memory (vector registers)
    __shared__ double ss[8 * 512];
    for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) ss[i] = out[64 + (i & 127)];
    __syncthreads();
    double x[8], a[8];
    const double *in = out + 64 + (threadIdx.x & 7) * 16;
    for (int k = 0; k < 8; ++k) { x[k] = in[k]; a[k] = in[8 + k]; }
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(x[k], ss[8 * (i & 511) + k], a[k]);
    }
    double r = 0; for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 1.2345) out[0] = r;
}
template <typename K>
void run(const char *name, K k) {
    double *o; cudaMalloc(&o, 8 * 4096);
    double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 0.5 + 1e-4 * (i % 97);
    cudaMemcpy(o, h, sizeof h, cudaMemcpyHostToDevice);
    static double hc[8 * ITERS]; for (int i = 0; i < 8 * ITERS; ++i) hc[i] = 0.99 + 1e-6 * (i % 13);
    cudaMemcpyToSymbol(cs, hc, sizeof hc);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k<<<sms * 4, 256>>>(o);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); for (int r = 0; r < 20; ++r) k<<<sms * 4, 256>>>(o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 20.0 * sms * 4 * 256 * ITERS * 8 * 2;
    printf("%s: %.2f TFLOP/s %s\n", name, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() { run("uniform (const) operand", kU); run("shared (vector) operand", kS); }
