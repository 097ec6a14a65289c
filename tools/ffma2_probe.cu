// FP32 issue-rate probe: 3-register FFMA vs packed FFMA2 (fma.rn.f32x2),
// 8 independent chains per thread, 4 warps/SMSP.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_k(float *out, int iters, float a, float b) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    float y[8], z[8];
    for (int k = 0; k < 8; ++k) { y[k] = a + k * 1e-6f; z[k] = b + k * 1e-5f; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], y[k], z[k]);   // 3 distinct registers
    }
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_k(float2 *out, int iters, float a, float b) {
    float2 x[8];
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    float2 y[8], z[8];
    for (int k = 0; k < 8; ++k) {
        y[k] = make_float2(a + k * 1e-6f, a * 0.5f);
        z[k] = make_float2(b + k * 1e-5f, b * 0.25f);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], y[k], z[k]);
    }
    float2 s = make_float2(0.f, 0.f);
    for (int k = 0; k < 8; ++k) { s.x += x[k].x; s.y += x[k].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 512, iters = 1 << 16;
    float *o;
    cudaMalloc(&o, sizeof(float2) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ffma_k<<<blocks, threads>>>(o, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("FFMA  3-reg : %.1f TFLOP/s\n", fl / ms / 1e9);
        cudaEventRecord(e0);
        ffma2_k<<<blocks, threads>>>((float2 *)o, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2 packed: %.1f TFLOP/s\n", 2 * fl / ms / 1e9);
    }
    return 0;
}
