// FP32 pipe probe 2: does packed FFMA2 (fma.rn.f32x2) lose issue rate when its
// three 64-bit sources are distinct register pairs (as DFMA does on sm_100a)?
// Variants, 8 independent chains per thread, 16 warps/SM resident x 4 CTAs:
//   0  FFMA   x = x*y_k + z_k      (3 distinct 32-bit registers)
//   1  FFMA2  x = x*y_k + z_k      (3 distinct register pairs)
//   2  FFMA2  x = x*y   + z_k      (y shared by the 8 chains: reuse cache)
//   3  FFMA2  x = x*x   + z_k      (2 distinct)
//   4  FFMA2  x = x*y   + z        (y, z shared)
//   5  FMUL2 / FADD2 alternating   (2-source packed ops, independent chains)
//   6  FFMA2  x = x*y_k.F32 + z_k  (one operand a broadcast 32-bit register)
//   7  FFMA2 3-distinct alternating with FMUL2
//   8  two scalar 3-distinct FFMAs alternating with one FFMA2 x*x+z
//   9  FFMA2  x = x*y_k.F32 + z_k.F32
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_probe2 ffma2_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(512) probe(float2 *out, int iters, float a, float b) {
    float2 x[8], y[8], z[8];
    for (int k = 0; k < 8; ++k) {
        x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
        y[k] = make_float2(a + k * 1e-6f, a - k * 1e-6f);
        z[k] = make_float2(b + k * 1e-5f, b * 0.25f + k * 1e-5f);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (V == 0) {
                x[k].x = fmaf(x[k].x, y[k].x, z[k].x);
                x[k].y = fmaf(x[k].y, y[k].y, z[k].y);
            } else if (V == 1) {
                x[k] = __ffma2_rn(x[k], y[k], z[k]);
            } else if (V == 2) {
                x[k] = __ffma2_rn(x[k], y[0], z[k]);
            } else if (V == 3) {
                x[k] = __ffma2_rn(x[k], x[k], z[k]);
            } else if (V == 4) {
                x[k] = __ffma2_rn(x[k], y[0], z[0]);
            } else if (V == 5) {
                x[k] = (k & 1) ? __fadd2_rn(x[k], z[k]) : __fmul2_rn(x[k], y[k]);
            } else if (V == 6) {   // one 32-bit broadcast operand (R.F32 form)
                x[k] = __ffma2_rn(x[k], make_float2(y[k].x, y[k].x), z[k]);
            } else if (V == 7) {   // 3-distinct FFMA2 alternating with 2-source FMUL2
                x[k] = (k & 1) ? __fmul2_rn(x[k], y[k]) : __ffma2_rn(x[k], y[k], z[k]);
            } else if (V == 8) {   // scalar 3-distinct FFMA pairs alternating with FFMA2 x*x+z
                if (k & 1) {
                    x[k] = __ffma2_rn(x[k], x[k], z[k]);
                } else {
                    x[k].x = fmaf(x[k].x, y[k].x, z[k].x);
                    x[k].y = fmaf(x[k].y, y[k].y, z[k].y);
                }
            } else {               // two 32-bit broadcast operands
                x[k] = __ffma2_rn(x[k], make_float2(y[k].x, y[k].x), make_float2(z[k].y, z[k].y));
            }
        }
    }
    float2 s = make_float2(0.f, 0.f);
    for (int k = 0; k < 8; ++k) { s.x += x[k].x; s.y += x[k].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
static void run(const char *name, float2 *o, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<V><<<blocks, threads>>>(o, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // lane-FMAs per second (one packed instruction = 2 lanes)
    const double lanefma = 2.0 * 8 * iters * (double)blocks * threads;
    printf("%-34s %.2f T lane-FMA/s (%.1f TFLOP/s)\n", name, lanefma / best / 1e9, 2 * lanefma / best / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 512, iters = 1 << 15;
    float2 *o;
    cudaMalloc(&o, sizeof(float2) * blocks * threads);
    run<0>("FFMA  3 distinct", o, blocks, threads, iters);
    run<1>("FFMA2 3 distinct pairs", o, blocks, threads, iters);
    run<2>("FFMA2 shared multiplier", o, blocks, threads, iters);
    run<3>("FFMA2 x*x+z", o, blocks, threads, iters);
    run<4>("FFMA2 shared multiplier+addend", o, blocks, threads, iters);
    run<5>("FMUL2 / FADD2 alternating", o, blocks, threads, iters);
    run<6>("FFMA2 pair * R.F32 + pair", o, blocks, threads, iters);
    run<7>("FFMA2 3 distinct / FMUL2 alternating", o, blocks, threads, iters);
    run<8>("2 FFMA 3 distinct / FFMA2 x*x+z", o, blocks, threads, iters);
    run<9>("FFMA2 pair * R.F32 + R.F32", o, blocks, threads, iters);
    return 0;
}
