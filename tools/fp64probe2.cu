// rsqrt seed alternatives: MUFU.RSQ64H vs FP32 MUFU.RSQ via integer exponent rebias
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__device__ __forceinline__ double seed64(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double seed32(double x) {
    const int hi = __double2hiint(x);
    const float xf = __int_as_float((hi - (896 << 20)) << 3);
    float g; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(xf));
    return __hiloint2double((__float_as_int(g) >> 3) + (896 << 20), 0);
}
template <int MODE>
__global__ void k(double *out, double s) {
    double a[8]; const double b = 0.999999999, c = 1e-10;
    double z = s + threadIdx.x * 1e-9 + 1.0;
    for (int k2 = 0; k2 < 8; ++k2) a[k2] = s + k2 + threadIdx.x * 1e-9;
    for (int i = 0; i < ITERS; ++i) {
        double r = MODE ? seed32(z) : seed64(z);
        z = z + r * 1e-30;
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) a[k2] = fma(a[k2], b, c);
    }
    double r = z; for (int k2 = 0; k2 < 8; ++k2) r += a[k2];
    if (r == 1.2345) out[0] = r;
}
// accuracy of both seeds after the cubic correction
__global__ void acc(double *err, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    double x = exp(-55.0 + 110.0 * (i + 0.5) / n);  // 1e-24 .. 1e24
    double ref = 1.0 / sqrt(x);
    for (int m = 0; m < 2; ++m) {
        double y0 = m ? seed32(x) : seed64(x);
        double e0 = fabs(y0 - ref) / ref;
        double y2 = y0 * y0, e = fma(-x, y2, 1.0), p = fma(e, 0.375, 0.5);
        double y = fma(p, y0 * e, y0);
        double e1 = fabs(y - ref) / ref;
        atomicMax((unsigned long long *)&err[2 * m], __double_as_longlong(e0));
        atomicMax((unsigned long long *)&err[2 * m + 1], __double_as_longlong(e1));
    }
}
template <typename K>
float run(K kk) {
    double *o; cudaMalloc(&o, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    kk<<<sms * 8, 256>>>(o, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kk<<<sms * 8, 256>>>(o, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); cudaFree(o); return ms;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double fl = sms * 8 * 256.0 * ITERS * 8 * 2;
    printf("rsq64h seed + 8 dfma: %.2f TFLOP/s\n", fl / run(k<0>) / 1e9);
    printf("f32 rsq seed + 8 dfma: %.2f TFLOP/s\n", fl / run(k<1>) / 1e9);
    double *e; cudaMalloc(&e, 32); cudaMemset(e, 0, 32);
    acc<<<4096, 256>>>(e, 4096 * 256);
    double h[4]; cudaMemcpy(h, e, 32, cudaMemcpyDeviceToHost);
    printf("seed64 max rel err %.3e -> cubic %.3e\nseed32 max rel err %.3e -> cubic %.3e\n", h[0], h[1], h[2], h[3]);
}
