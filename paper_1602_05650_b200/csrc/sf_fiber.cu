// sf_fiber.cu — batched per-fiber self terms and the near-field correction
// apply (sm_100a).  These are HBM-bound small dense operations; the roofline
// is bytes of K / W read once per application.
#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

// kernels.py:284-334, one CTA per fiber.  Uses explicitly rounded operations
// (no FMA contraction) in the reference's evaluation order so that K is
// bitwise identical to the reference's numba build.
__global__ void kdelta_build_kernel(const double *__restrict__ X, const double *__restrict__ s,
                                    const double *__restrict__ s_alpha,
                                    const double *__restrict__ tang, const double *__restrict__ w,
                                    int n, const double *__restrict__ delta, double pref,
                                    double *__restrict__ K) {
    extern __shared__ double sh[];
    double *xs = sh;          // 3n
    double *ss = xs + 3 * n;  // n
    double *cw = ss + n;      // n
    const int m = blockIdx.x;
    const double *Xm = X + (int64_t)3 * n * m;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        xs[3 * j] = Xm[3 * j];
        xs[3 * j + 1] = Xm[3 * j + 1];
        xs[3 * j + 2] = Xm[3 * j + 2];
        ss[j] = s[(int64_t)n * m + j];
        cw[j] = __dmul_rn(__dmul_rn(w[j], s_alpha[(int64_t)n * m + j]), pref);
    }
    __syncthreads();
    const double dl = delta[m];
    const double d2 = __dmul_rn(dl, dl);
    const int ld = 3 * n;
    double *Km = K + (int64_t)9 * n * n * m;
    // off-diagonal 3x3 blocks
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int i = idx / n, j = idx - (idx / n) * n;
        if (i == j) continue;
        const double rx = __dsub_rn(xs[3 * i], xs[3 * j]);
        const double ry = __dsub_rn(xs[3 * i + 1], xs[3 * j + 1]);
        const double rz = __dsub_rn(xs[3 * i + 2], xs[3 * j + 2]);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
        const double reg = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(r2, d2)));
        const double a = __dmul_rn(cw[j], reg);
        const double b = __ddiv_rn(__dmul_rn(cw[j], reg), r2);
        const double bx = __dmul_rn(b, rx), by = __dmul_rn(b, ry), bz = __dmul_rn(b, rz);
        double *r0 = Km + (int64_t)(3 * i) * ld + 3 * j;
        double *r1 = r0 + ld;
        double *r2p = r1 + ld;
        r0[0] = __dadd_rn(0.0, __dadd_rn(a, __dmul_rn(bx, rx)));
        r0[1] = __dadd_rn(0.0, __dmul_rn(bx, ry));
        r0[2] = __dadd_rn(0.0, __dmul_rn(bx, rz));
        r1[0] = __dadd_rn(0.0, __dmul_rn(by, rx));
        r1[1] = __dadd_rn(0.0, __dadd_rn(a, __dmul_rn(by, ry)));
        r1[2] = __dadd_rn(0.0, __dmul_rn(by, rz));
        r2p[0] = __dadd_rn(0.0, __dmul_rn(bz, rx));
        r2p[1] = __dadd_rn(0.0, __dmul_rn(bz, ry));
        r2p[2] = __dadd_rn(0.0, __dadd_rn(a, __dmul_rn(bz, rz)));
    }
    // diagonal blocks: the local subtraction, accumulated over j in order
    const double *Tm = tang + (int64_t)3 * n * m;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double tx = Tm[3 * i], ty = Tm[3 * i + 1], tz = Tm[3 * i + 2];
        const double xx = __dadd_rn(1.0, __dmul_rn(tx, tx));
        const double yy = __dadd_rn(1.0, __dmul_rn(ty, ty));
        const double zz = __dadd_rn(1.0, __dmul_rn(tz, tz));
        double d[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const double ds = __dsub_rn(ss[i], ss[j]);
            const double sub = __ddiv_rn(cw[j], __dsqrt_rn(__dadd_rn(__dmul_rn(ds, ds), d2)));
            const double sx = __dmul_rn(sub, tx), sy = __dmul_rn(sub, ty), sz = __dmul_rn(sub, tz);
            d[0] = __dsub_rn(d[0], __dmul_rn(sub, xx));
            d[1] = __dsub_rn(d[1], __dmul_rn(sx, ty));
            d[2] = __dsub_rn(d[2], __dmul_rn(sx, tz));
            d[3] = __dsub_rn(d[3], __dmul_rn(sy, tx));
            d[4] = __dsub_rn(d[4], __dmul_rn(sub, yy));
            d[5] = __dsub_rn(d[5], __dmul_rn(sy, tz));
            d[6] = __dsub_rn(d[6], __dmul_rn(sz, tx));
            d[7] = __dsub_rn(d[7], __dmul_rn(sz, ty));
            d[8] = __dsub_rn(d[8], __dmul_rn(sub, zz));
        }
        double *r0 = Km + (int64_t)(3 * i) * ld + 3 * i;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) r0[(int64_t)a * ld + b] = d[3 * a + b];
    }
}

int fiber_kdelta_build(const double *X, const double *s, const double *s_alpha,
                       const double *tang, const double *w, int64_t nf, int64_t n,
                       const double *delta, double pref, double *K, cudaStream_t st) {
    if (nf == 0) return SF_OK;
    const size_t smem = sizeof(double) * 5 * (size_t)n;
    kdelta_build_kernel<<<(unsigned)nf, 256, smem, st>>>(X, s, s_alpha, tang, w, (int)n, delta,
                                                         pref, K);
    return check_launch("kdelta_build_kernel");
}

// u = M f + K f (fiber.py:244-258).  One CTA per fiber, a warp per 4 K rows,
// lanes stride the rows (coalesced 256-byte reads), shuffle reductions.
__global__ void self_apply_kernel(const double *__restrict__ K, const double *__restrict__ tang,
                                  const double *__restrict__ c_log, double c_two,
                                  const double *__restrict__ f, int n, int accumulate,
                                  double *__restrict__ u) {
    extern __shared__ double fs[];  // 3n
    const int m = blockIdx.x;
    const int ld = 3 * n;
    const double *fm = f + (int64_t)ld * m;
    for (int c = threadIdx.x; c < ld; c += blockDim.x) fs[c] = fm[c];
    __syncthreads();
    const double *Km = K ? K + (int64_t)ld * ld * m : nullptr;
    const double *Tm = tang + (int64_t)ld * m;
    const double cl = c_log[m];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // 4 rows per warp pass: 4 independent coalesced K loads per lane in flight
    constexpr int RB = 4;
    for (int r0 = warp * RB; r0 < ld; r0 += nw * RB) {
        double accs[RB] = {0.0, 0.0, 0.0, 0.0};
        if (K) {   // K == nullptr: local mobility only
            for (int c = lane; c < ld; c += 32) {
                const double fc = fs[c];
#pragma unroll
                for (int q = 0; q < RB; ++q)
                    if (r0 + q < ld) accs[q] = fma(Km[(int64_t)(r0 + q) * ld + c], fc, accs[q]);
            }
#pragma unroll
            for (int q = 0; q < RB; ++q) accs[q] = warp_sum(accs[q]);
        }
        if (lane < RB && r0 + lane < ld) {
            const int r = r0 + lane;
            double acc = accs[0];
#pragma unroll
            for (int q = 1; q < RB; ++q) acc = lane == q ? accs[q] : acc;
            const int i = r / 3, a = r - 3 * (r / 3);
            const double tx = Tm[3 * i], ty = Tm[3 * i + 1], tz = Tm[3 * i + 2];
            const double fdt = fs[3 * i] * tx + fs[3 * i + 1] * ty + fs[3 * i + 2] * tz;
            const double ta = a == 0 ? tx : (a == 1 ? ty : tz);
            const double fa = fs[r];
            const double ft = fdt * ta;
            const double mob = cl * (fa + ft) + c_two * (fa - ft);
            const double v = mob + acc;
            double *dst = u + (int64_t)ld * m + r;
            *dst = accumulate ? *dst + v : v;
        }
    }
}

int fiber_self_apply(const double *K, const double *tang, const double *c_log, double c_two,
                     const double *f, int64_t nf, int64_t n, int accumulate, double *u,
                     cudaStream_t st) {
    if (nf == 0) return SF_OK;
    const size_t smem = sizeof(double) * 3 * (size_t)n;
    self_apply_kernel<<<(unsigned)nf, 256, smem, st>>>(K, tang, c_log, c_two, f, (int)n,
                                                       accumulate, u);
    return check_launch("self_apply_kernel");
}

// Near-field correction apply (system.py:702-707).  Warp per distinct target;
// entries applied in list order.
__global__ void near_apply_kernel(const int64_t *__restrict__ row_ptr,
                                  const int64_t *__restrict__ rows, int64_t nrows,
                                  const int64_t *__restrict__ w_off,
                                  const int64_t *__restrict__ x_off,
                                  const int64_t *__restrict__ x_len, const double *__restrict__ W,
                                  const double *__restrict__ x, double *__restrict__ u) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= nrows) return;
    const int64_t t = rows[gw];
    double u0 = 0, u1 = 0, u2 = 0;
    if (lane == 0) {
        u0 = u[3 * t]; u1 = u[3 * t + 1]; u2 = u[3 * t + 2];
    }
    for (int64_t e = row_ptr[gw]; e < row_ptr[gw + 1]; ++e) {
        const int64_t L = x_len[e];
        const double *We = W + w_off[e];
        const double *xe = x + x_off[e];
        double a0 = 0, a1 = 0, a2 = 0;
        for (int64_t c = lane; c < L; c += 32) {
            const double xv = xe[c];
            a0 = fma(We[c], xv, a0);
            a1 = fma(We[L + c], xv, a1);
            a2 = fma(We[2 * L + c], xv, a2);
        }
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
        a2 = warp_sum(a2);
        if (lane == 0) {
            u0 += a0; u1 += a1; u2 += a2;
        }
    }
    if (lane == 0) {
        u[3 * t] = u0; u[3 * t + 1] = u1; u[3 * t + 2] = u2;
    }
}

int near_apply(const int64_t *row_ptr, const int64_t *rows, int64_t nrows, const int64_t *w_off,
               const int64_t *x_off, const int64_t *x_len, const double *W, const double *x,
               double *u, cudaStream_t st) {
    if (nrows == 0) return SF_OK;
    const int64_t threads = nrows * 32;
    near_apply_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(row_ptr, rows, nrows,
                                                                        w_off, x_off, x_len, W,
                                                                        x, u);
    return check_launch("near_apply_kernel");
}

// Per-fiber geometry (spectral.py:139-154, fiber.py:133-147, 172-174):
// Xa = D X, s_alpha = |Xa|, t = Xa / s_alpha, s = S s_alpha (S integrates the
// interpolant from the minus end), L = s[0], node weights w_cc * s_alpha,
// delta = ratio * L when ratio > 0.  One CTA per fiber.
__global__ void geometry_kernel(const double *__restrict__ X, int n, const double *__restrict__ D,
                                const double *__restrict__ S, const double *__restrict__ wcc,
                                double delta_ratio, double *__restrict__ s,
                                double *__restrict__ s_alpha, double *__restrict__ tang,
                                double *__restrict__ wnode, double *__restrict__ L,
                                double *__restrict__ delta, int *__restrict__ degenerate) {
    extern __shared__ double sh[];
    double *xs = sh;          // 3n
    double *sa = xs + 3 * n;  // n
    const int m = blockIdx.x;
    const int64_t base = (int64_t)n * m;
    for (int j = threadIdx.x; j < 3 * n; j += blockDim.x) xs[j] = X[3 * base + j];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double ax = 0, ay = 0, az = 0;
        for (int j = 0; j < n; ++j) {
            const double d = D[(int64_t)i * n + j];
            ax = fma(d, xs[3 * j], ax);
            ay = fma(d, xs[3 * j + 1], ay);
            az = fma(d, xs[3 * j + 2], az);
        }
        const double v = sqrt(ax * ax + ay * ay + az * az);
        sa[i] = v;
        if (!(v > 1e-12)) atomicAdd(degenerate, 1);
        s_alpha[base + i] = v;
        tang[3 * (base + i)] = ax / v;
        tang[3 * (base + i) + 1] = ay / v;
        tang[3 * (base + i) + 2] = az / v;
        wnode[base + i] = wcc[i] * v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double acc = 0;
        for (int j = 0; j < n; ++j) acc = fma(S[(int64_t)i * n + j], sa[j], acc);
        s[base + i] = acc;
        if (i == 0) {
            L[m] = acc;
            if (delta_ratio > 0) delta[m] = delta_ratio * acc;
        }
    }
}

int fiber_geometry(const double *X, int64_t nf, int64_t n, const double *D, const double *S,
                   const double *wcc, double delta_ratio, double *s, double *s_alpha,
                   double *tang, double *wnode, double *L, double *delta, int *degenerate,
                   cudaStream_t st) {
    if (nf == 0) return SF_OK;
    if (degenerate && cudaMemsetAsync(degenerate, 0, sizeof(int), st) != cudaSuccess)
        return check_launch("memset");
    const size_t smem = sizeof(double) * 4 * (size_t)n;
    geometry_kernel<<<(unsigned)nf, 128, smem, st>>>(X, (int)n, D, S, wcc, delta_ratio, s,
                                                     s_alpha, tang, wnode, L, delta, degenerate);
    return check_launch("geometry_kernel");
}

}  // namespace sf
