// sf_near.cu — device construction of the fiber near-field correction maps
// (SURVEY.md §8f rank 1): the candidate search of InteractionCache
// (system.py:564-586) and near_fiber_weights - plain_fiber_weights
// (fiber.py:453-575) for every (target, fiber) pair inside the near shell.
//
// One CTA per pair: Chebyshev coefficients of the centreline and of s_alpha,
// nearest centreline point (8p+1 samples, then 50 golden-section steps as the
// reference does), adaptive bisection into 10-point Gauss-Legendre panels
// until each is shorter than its distance to the target (depth <= 14), panel
// quadrature of the Stokeslet (+ doublet) kernel resampled to the nodal
// density by barycentric rows, smoothstep blend to the plain collocation sum
// near the shell boundary, and finally W_near - W_plain (3 x 3n).
#include <cmath>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

constexpr int kNearThreads = 128;
constexpr int kMaxPanels = 512;

struct NearArgs {
    const int64_t *pt, *pl;      // pair target index, fiber index
    const double *targets;       // (nt,3)
    const double *X;             // (nf,n,3)
    const double *s_alpha;       // (nf,n)
    const double *wcc;           // (n) Clenshaw-Curtis weights
    const double *Cmat;          // (n,n) nodal values -> Chebyshev coefficients
    const double *nodes;         // (n)
    const double *gl;            // 10 GL nodes then 10 weights on [-1,1]
    const double *eps, *L;       // (nf)
    int n;
    double mu;
    int include_doublet;
    double *W;                   // (npairs, 3, 3n)
    int *info;                   // (npairs): 0 ok, 1 inside fiber, 2 panel overflow
};

// numpy.polynomial.chebyshev.chebval recurrence (Clenshaw), coefficients c[0..n)
__device__ double clenshaw(const double *c, int n, double x) {
    if (n == 1) return c[0];
    double c0, c1;
    if (n == 2) {
        c0 = c[0];
        c1 = c[1];
    } else {
        const double x2 = 2.0 * x;
        c0 = c[n - 2];
        c1 = c[n - 1];
        for (int i = 3; i <= n; ++i) {
            const double tmp = c0;
            c0 = c[n - i] - c1;
            c1 = tmp + c1 * x2;
        }
    }
    return c0 + c1 * x;
}

__device__ void kernel_block(double rx, double ry, double rz, int dbl, double coeff, double *K) {
    const double d2 = rx * rx + ry * ry + rz * rz;
    const double d = sqrt(d2);
    const double r[3] = {rx, ry, rz};
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            const double rr = r[a] * r[b];
            const double e = (a == b) ? 1.0 : 0.0;
            double k = e / d + rr / (d2 * d);
            if (dbl) k += coeff * (e / (d2 * d) - 3.0 * rr / (d2 * d2 * d));
            K[3 * a + b] = k;
        }
}

__global__ void __launch_bounds__(kNearThreads) near_weights_kernel(NearArgs A) {
    const int n = A.n, p = n - 1, tid = threadIdx.x;
    const int64_t e = blockIdx.x;
    const int64_t t = A.pt[e], l = A.pl[e];
    extern __shared__ double sm[];
    double *cx = sm;                  // 3n coefficients
    double *csa = cx + 3 * n;         // n
    double *Xl = csa + n;             // 3n nodal positions
    double *qK = Xl + 3 * n;          // kNearThreads x 9
    double *qc = qK + 9 * kNearThreads;   // kNearThreads: w * s_alpha
    double *qinv = qc + kNearThreads;     // kNearThreads: 1 / sum_j t_j
    double *qal = qinv + kNearThreads;    // kNearThreads: alpha
    int *qhit = (int *)(qal + kNearThreads);             // kNearThreads
    double *pa = (double *)(qhit + kNearThreads);        // kMaxPanels
    double *pb = pa + kMaxPanels;                        // kMaxPanels
    __shared__ double s_red[kNearThreads];
    __shared__ int s_idx[kNearThreads];
    __shared__ double s_wb;
    __shared__ int s_np, s_fail;

    const double tx = A.targets[3 * t], ty = A.targets[3 * t + 1], tz = A.targets[3 * t + 2];
    const double *X = A.X + (int64_t)3 * n * l;
    const double *sa = A.s_alpha + (int64_t)n * l;
    for (int k = tid; k < 3 * n; k += blockDim.x) Xl[k] = X[k];
    __syncthreads();
    for (int k = tid; k < 4 * n; k += blockDim.x) {
        const int comp = k / n, row = k - comp * n;
        double acc = 0.0;
        for (int j = 0; j < n; ++j)
            acc += A.Cmat[row * n + j] * (comp < 3 ? Xl[3 * j + comp] : sa[j]);
        if (comp < 3) cx[comp * n + row] = acc;
        else csa[row] = acc;
    }
    __syncthreads();

    // ---- nearest centreline point (fiber.py:453-481)
    const int ns = 8 * p + 1;
    const double step = M_PI / (double)(ns - 1);
    double best = 1e300;
    int bi = 0x7fffffff;
    for (int k = tid; k < ns; k += blockDim.x) {
        const double al = cos((double)k * step);
        const double dx = clenshaw(cx, n, al) - tx, dy = clenshaw(cx + n, n, al) - ty,
                     dz = clenshaw(cx + 2 * n, n, al) - tz;
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        if (d2 < best || (d2 == best && k < bi)) { best = d2; bi = k; }
    }
    s_red[tid] = best;
    s_idx[tid] = bi;
    __syncthreads();
    if (tid == 0) {
        for (int k = 1; k < blockDim.x; ++k)
            if (s_red[k] < best || (s_red[k] == best && s_idx[k] < bi)) { best = s_red[k]; bi = s_idx[k]; }
        const int i0 = bi;
        double lo = cos((double)min(i0 + 1, ns - 1) * step);
        double hi = cos((double)max(i0 - 1, 0) * step);
        auto d2_at = [&](double a) {
            const double dx = clenshaw(cx, n, a) - tx, dy = clenshaw(cx + n, n, a) - ty,
                         dz = clenshaw(cx + 2 * n, n, a) - tz;
            return (dx * dx + dy * dy) + dz * dz;
        };
        for (int it = 0; it < 50; ++it) {
            const double m1 = lo + 0.382 * (hi - lo), m2 = lo + 0.618 * (hi - lo);
            if (d2_at(m1) < d2_at(m2)) hi = m2;
            else lo = m1;
        }
        const double a0 = 0.5 * (lo + hi);
        const double dx = tx - clenshaw(cx, n, a0), dy = ty - clenshaw(cx + n, n, a0),
                     dz = tz - clenshaw(cx + 2 * n, n, a0);
        const double d = sqrt(dx * dx + dy * dy + dz * dz);
        const double Lf = A.L[l];
        s_fail = d < A.eps[l] * Lf ? 1 : 0;
        // ---- adaptive panels (fiber.py:535-549), LIFO as the reference
        int np_ = 0;
        double stk_a[64], stk_b[64];
        int stk_d[64];
        int top = 1;
        stk_a[0] = -1.0; stk_b[0] = 1.0; stk_d[0] = 0;
        while (top > 0 && !s_fail) {
            --top;
            const double a = stk_a[top], b = stk_b[top];
            const int depth = stk_d[top];
            const double pr[3] = {a, 0.5 * (a + b), b};
            double dmin2 = 1e300;
            for (int q = 0; q < 3; ++q) {
                const double ex = clenshaw(cx, n, pr[q]) - tx, ey = clenshaw(cx + n, n, pr[q]) - ty,
                             ez = clenshaw(cx + 2 * n, n, pr[q]) - tz;
                dmin2 = fmin(dmin2, (ex * ex + ey * ey) + ez * ez);
            }
            const double dmin = sqrt(dmin2);
            if (0.5 * (b - a) * Lf > dmin && depth < 14) {
                if (top + 2 > 64) { s_fail = 2; break; }
                const double mid = 0.5 * (a + b);
                stk_a[top] = a; stk_b[top] = mid; stk_d[top] = depth + 1; ++top;
                stk_a[top] = mid; stk_b[top] = b; stk_d[top] = depth + 1; ++top;
                continue;
            }
            if (np_ >= kMaxPanels) { s_fail = 2; break; }
            pa[np_] = a;
            pb[np_] = b;
            ++np_;
        }
        s_np = np_;
        const double shell = 1.5 * Lf / p;
        const double xb = (d - 0.8 * shell) / (0.2 * shell);
        if (xb > 0.0) {
            const double xm = fmin(xb, 1.0);
            s_wb = xm * xm * (3.0 - 2.0 * xm);
        } else {
            s_wb = -1.0;
        }
    }
    __syncthreads();
    if (s_fail) {
        if (tid == 0) A.info[e] = s_fail;
        return;
    }
    const int nq = 10 * s_np;
    const double coeff = A.eps[l] * A.L[l];
    const double dco = coeff * coeff / 2.0;
    // barycentric weights of the Chebyshev nodes
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const int j = tid;
    const double wj = (j < n) ? ((j % 2 ? -1.0 : 1.0) * ((j == 0 || j == n - 1) ? 0.5 : 1.0)) : 0.0;
    const double nodej = (j < n) ? A.nodes[j] : 0.0;
    for (int base = 0; base < nq; base += kNearThreads) {
        const int q = base + tid;
        if (q < nq) {
            const int pi = q / 10, k = q - 10 * pi;
            const double a = pa[pi], b = pb[pi];
            const double al = 0.5 * (a + b) + 0.5 * (b - a) * A.gl[k];
            const double wq = 0.5 * (b - a) * A.gl[10 + k];
            const double xp = clenshaw(cx, n, al), yp = clenshaw(cx + n, n, al),
                         zp = clenshaw(cx + 2 * n, n, al);
            const double sq = clenshaw(csa, n, al);
            kernel_block(tx - xp, ty - yp, tz - zp, A.include_doublet, dco, qK + 9 * tid);
            qc[tid] = wq * sq;
            qal[tid] = al;
            // barycentric row normaliser; exact node hits give an indicator row
            double sum = 0.0;
            int hit = -1;
            for (int jj = 0; jj < n; ++jj) {
                const double dd = al - A.nodes[jj];
                const double wjj = (jj % 2 ? -1.0 : 1.0) * ((jj == 0 || jj == n - 1) ? 0.5 : 1.0);
                if (fabs(dd) < 1e-14) {
                    if (hit < 0) hit = jj;
                    sum += wjj / 1.0;
                } else {
                    sum += wjj / dd;
                }
            }
            qinv[tid] = sum;
            qhit[tid] = hit;
        }
        __syncthreads();
        const int cnt = min(kNearThreads, nq - base);
        if (j < n) {
            for (int qq = 0; qq < cnt; ++qq) {
                double P;
                if (qhit[qq] >= 0) {
                    P = (j == qhit[qq]) ? 1.0 : 0.0;
                } else {
                    const double dd = qal[qq] - nodej;
                    P = (wj / dd) / qinv[qq];
                }
                const double cP = qc[qq] * P;
#pragma unroll
                for (int ab = 0; ab < 9; ++ab) acc[ab] = fma(cP, qK[9 * qq + ab], acc[ab]);
            }
        }
        __syncthreads();
    }
    if (j < n) {
        const double inv = 1.0 / (8.0 * M_PI * A.mu);
        // plain collocation weights at node j (fiber.py:568-575)
        double Kp[9];
        kernel_block(tx - Xl[3 * j], ty - Xl[3 * j + 1], tz - Xl[3 * j + 2], A.include_doublet, dco,
                     Kp);
        const double wn = A.wcc[j] * A.s_alpha[(int64_t)n * l + j];
        double *out = A.W + (int64_t)e * 9 * n;
        const double wb = s_wb;
        for (int aa = 0; aa < 3; ++aa)
            for (int bb = 0; bb < 3; ++bb) {
                const double wnear = acc[3 * aa + bb] * inv;
                const double wplain = wn * Kp[3 * aa + bb] * inv;
                const double w = wb > 0.0 ? (1.0 - wb) * wnear + wb * wplain : wnear;
                out[(int64_t)aa * 3 * n + 3 * j + bb] = w - wplain;
            }
    }
    if (tid == 0) A.info[e] = 0;
}

// Candidate search: for every target t and fiber l != group(t) with the
// minimum node distance below the fiber's shell (system.py:566-577).  A
// bounding-sphere test prunes; hits are appended (order fixed later).
__global__ void near_search_kernel(const double *__restrict__ trg, const int64_t *__restrict__ tgrp,
                                   int64_t nt, const double *__restrict__ X, int n, int64_t nf,
                                   const double *__restrict__ center, const double *__restrict__ bound,
                                   const double *__restrict__ shell, unsigned long long *count,
                                   int64_t *pairs, int64_t cap) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double x = trg[3 * t], y = trg[3 * t + 1], z = trg[3 * t + 2];
        const int64_t g = tgrp ? tgrp[t] : -1;
        for (int64_t l = 0; l < nf; ++l) {
            if (g == l) continue;
            const double cx = x - center[3 * l], cy = y - center[3 * l + 1], cz = z - center[3 * l + 2];
            const double bb = bound[l];
            if (cx * cx + cy * cy + cz * cz > bb * bb) continue;
            const double sh = shell[l];
            const double *Xl = X + (int64_t)3 * n * l;
            double d2min = 1e300;
            for (int k = 0; k < n; ++k) {
                const double dx = x - Xl[3 * k], dy = y - Xl[3 * k + 1], dz = z - Xl[3 * k + 2];
                d2min = fmin(d2min, dx * dx + dy * dy + dz * dz);
            }
            if (d2min < sh * sh) {
                const unsigned long long slot = atomicAdd(count, 1ull);
                if ((int64_t)slot < cap) {
                    pairs[2 * slot] = l;
                    pairs[2 * slot + 1] = t;
                }
            }
        }
    }
}

}  // namespace sf

using namespace sf;

extern "C" int sf_near_search(const double *trg, const int64_t *tgrp, int64_t nt, const double *X,
                              int64_t nf, int64_t n, const double *center, const double *bound,
                              const double *shell, int64_t cap, int64_t *pairs,
                              unsigned long long *count, void *stream) {
    if (nt < 0 || nf < 0 || n < 2 || cap < 0) return set_error(SF_EINVAL, "bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), st) != cudaSuccess)
        return check_launch("memset");
    if (nt == 0 || nf == 0) return SF_OK;
    int64_t blocks = (nt + 127) / 128;
    if (blocks > 8192) blocks = 8192;
    near_search_kernel<<<(unsigned)blocks, 128, 0, st>>>(trg, tgrp, nt, X, (int)n, nf, center,
                                                         bound, shell, count, pairs, cap);
    return check_launch("near_search_kernel");
}

extern "C" int sf_near_fiber_weights(const int64_t *pt, const int64_t *pl, int64_t npairs,
                                     const double *targets, const double *X, const double *s_alpha,
                                     const double *wcc, const double *Cmat, const double *nodes,
                                     const double *gl, const double *eps, const double *L,
                                     int64_t n, double mu, int include_doublet, double *W,
                                     int *info, void *stream) {
    if (npairs < 0 || n < 5 || n > kNearThreads) return set_error(SF_EINVAL, "bad sizes");
    if (npairs == 0) return SF_OK;
    NearArgs A{pt, pl, targets, X, s_alpha, wcc, Cmat, nodes, gl, eps, L, (int)n, mu,
               include_doublet, W, info};
    const size_t smem = sizeof(double) * (7 * n + 12 * kNearThreads + 2 * kMaxPanels) +
                        sizeof(int) * kNearThreads + 64;
    if (cudaFuncSetAttribute(near_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    near_weights_kernel<<<(unsigned)npairs, kNearThreads, smem, (cudaStream_t)stream>>>(A);
    return check_launch("near_weights_kernel");
}

// ---------------------------------------------------------------------------
// Near-surface correction maps on the device (body.py:371-519 via
// system.py:588-613): for each (target, surface) pair
//   W = B^T [ ell_0 (P(x0) - RS (x) r0 + jump I (x) r0) + sum_k ell_k P(pt_k) ]
//       - P_coarse(target)
// where P(y) is the stresslet quadrature map of the upsampled ("fine") mesh
// at the point y, RS the row sum of P(x0) over the fine nodes, r0 the fine
// interpolation row at the nearest surface point (theta0, phi0), ell the
// Lagrange weights of the off-surface extrapolation points and B the
// fine-from-coarse patch interpolation.  The host supplies the per-pair
// scalars (nearest point by the reference's golden-section search, ell,
// pt_k, r0); the device does every O(N_fine) sum.  One CTA per (coarse
// patch, pair): it evaluates the f*f*16 fine nodes inside its coarse patch
// into shared memory and contracts them with their interpolation
// coefficients in a fixed order (no atomics), so results are reproducible.
namespace sf {
namespace {
constexpr int kSurfRsBlocks = 148, kSurfThreads = 160;

struct SurfArgs {
    const double *cnodes, *cnrm, *cw;   // coarse mesh (patch-major, 16 nodes per patch)
    int64_t nt, nph;                    // coarse patch grid
    const double *fnodes, *fnrm, *fw;   // fine mesh, patch grid (f nt, f nph)
    const double *fcoef;                // (Nf, 8): cu[4], cv[4] of each fine node in its coarse patch
    int f;
    int64_t npairs;
    const double *trg, *x0, *pts, *ell, *jump, *r0coef;   // (np,3) (np,3) (np,3,3) (np,4) (np) (np,16)
    const int64_t *r0patch;             // (np) fine patch index of (theta0, phi0)
    double pref;                        // -3 / (4 pi mu)
    double *rs;                         // (np, 9) work: row sums
    double *rs_part;                    // (np, kSurfRsBlocks, 9)
    double *W;                          // (np, 3, 3 Nc)
};

__device__ __forceinline__ void plain_at(const double *y, const double *node, const double *nrm,
                                         double w, double pref, double s[9]) {
    const double r0 = y[0] - node[0], r1 = y[1] - node[1], r2 = y[2] - node[2];
    const double d2 = r0 * r0 + r1 * r1 + r2 * r2;
    double sc = 0.0;
    if (d2 > 1e-24) {
        const double nr = nrm[0] * r0 + nrm[1] * r1 + nrm[2] * r2;
        sc = pref * w * nr / (d2 * d2 * sqrt(d2));
    }
    const double r[3] = {r0, r1, r2};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) s[3 * a + b] = sc * r[a] * r[b];
}

__global__ void surf_rs_partial(SurfArgs A, int64_t nf) {
    const int64_t p = blockIdx.y;
    const double *y = A.x0 + 3 * p;
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < nf;
         m += (int64_t)gridDim.x * blockDim.x) {
        double s[9];
        plain_at(y, A.fnodes + 3 * m, A.fnrm + 3 * m, A.fw[m], A.pref, s);
#pragma unroll
        for (int e = 0; e < 9; ++e) acc[e] += s[e];
    }
    __shared__ double red[9][kSurfThreads / 32];
#pragma unroll
    for (int e = 0; e < 9; ++e) {
        const double v = warp_sum(acc[e]);
        if ((threadIdx.x & 31) == 0) red[e][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        double v = 0.0;
        for (int k = 0; k < kSurfThreads / 32; ++k) v += red[threadIdx.x][k];
        A.rs_part[(p * kSurfRsBlocks + blockIdx.x) * 9 + threadIdx.x] = v;
    }
}

__global__ void surf_rs_final(SurfArgs A) {
    const int64_t p = blockIdx.x;
    if (threadIdx.x < 9) {
        double v = 0.0;
        for (int k = 0; k < kSurfRsBlocks; ++k) v += A.rs_part[(p * kSurfRsBlocks + k) * 9 + threadIdx.x];
        A.rs[p * 9 + threadIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kSurfThreads) surf_patch_kernel(SurfArgs A) {
    extern __shared__ double sm[];
    const int f = A.f, nloc = f * f * 16;
    double *Wf = sm;                    // nloc x 9
    double *cf = sm + 9 * nloc;         // nloc x 8
    const int64_t P = blockIdx.x, p = blockIdx.y;
    const int64_t it = P / A.nph, ip = P - it * A.nph;
    const int64_t nphf = A.nph * f;
    const double *x0 = A.x0 + 3 * p, *pts = A.pts + 9 * p, *ell = A.ell + 4 * p;
    const double jump = A.jump[p];
    const int64_t r0p = A.r0patch[p];
    double RS[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) RS[e] = A.rs[p * 9 + e];
    for (int ml = threadIdx.x; ml < nloc; ml += blockDim.x) {
        const int fl = ml >> 4, q = ml & 15;
        const int64_t ft = it * f + fl / f, fp = ip * f + fl % f;
        const int64_t fpatch = ft * nphf + fp;
        const int64_t m = fpatch * 16 + q;
        const double *node = A.fnodes + 3 * m, *nrm = A.fnrm + 3 * m;
        const double w = A.fw[m];
        double s0[9], sk[9], out[9];
        plain_at(x0, node, nrm, w, A.pref, s0);
        const double r0 = fpatch == r0p ? A.r0coef[p * 16 + q] : 0.0;
#pragma unroll
        for (int e = 0; e < 9; ++e) {
            double v = s0[e] - RS[e] * r0;
            if (e % 4 == 0) v += jump * r0;
            out[e] = ell[0] * v;
        }
#pragma unroll
        for (int k = 1; k < 4; ++k) {
            if (ell[k] == 0.0) continue;
            plain_at(pts + 3 * (k - 1), node, nrm, w, A.pref, sk);
#pragma unroll
            for (int e = 0; e < 9; ++e) out[e] += ell[k] * sk[e];
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) Wf[ml * 9 + e] = out[e];
#pragma unroll
        for (int e = 0; e < 8; ++e) cf[ml * 8 + e] = A.fcoef[m * 8 + e];
    }
    __syncthreads();
    if (threadIdx.x < 144) {
        const int n = threadIdx.x / 9, e = threadIdx.x - 9 * n;
        const int un = n >> 2, vn = n & 3;
        double acc = 0.0;
        for (int ml = 0; ml < nloc; ++ml) acc += (cf[ml * 8 + un] * cf[ml * 8 + 4 + vn]) * Wf[ml * 9 + e];
        const int64_t cn = (it * A.nph + ip) * 16 + n;
        double sp[9];
        plain_at(A.trg + 3 * p, A.cnodes + 3 * cn, A.cnrm + 3 * cn, A.cw[cn], A.pref, sp);
        acc -= sp[e];
        const int a = e / 3, b = e - 3 * a;
        const int64_t Nc = A.nt * A.nph * 16;
        A.W[(p * 3 + a) * 3 * Nc + 3 * cn + b] = acc;
    }
}
}  // namespace

}  // namespace sf

extern "C" int sf_near_surface_weights(
    const double *cnodes, const double *cnrm, const double *cw, int64_t nt, int64_t nph,
    const double *fnodes, const double *fnrm, const double *fw, const double *fcoef, int f,
    int64_t npairs, const double *trg, const double *x0, const double *pts, const double *ell,
    const double *jump, const int64_t *r0patch, const double *r0coef, double mu, double *work,
    double *W, void *stream) {
    using namespace sf;
    if (npairs <= 0) return SF_OK;
    if (nt < 1 || nph < 1 || f < 1 || f > 8) return set_error(SF_EINVAL, "bad patch grid");
    if (!cnodes || !cnrm || !cw || !fnodes || !fnrm || !fw || !fcoef || !trg || !x0 || !pts ||
        !ell || !jump || !r0patch || !r0coef || !work || !W)
        return set_error(SF_EINVAL, "null pointer");
    if (!(mu > 0)) return set_error(SF_EINVAL, "viscosity must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    // pairs ride gridDim.y (<= 65535): launch in chunks
    constexpr int64_t kChunk = 65535;
    if (npairs > kChunk) {
        const int64_t Nc = nt * nph * 16;
        for (int64_t p0 = 0; p0 < npairs; p0 += kChunk) {
            const int64_t k = npairs - p0 < kChunk ? npairs - p0 : kChunk;
            const int rc = sf_near_surface_weights(
                cnodes, cnrm, cw, nt, nph, fnodes, fnrm, fw, fcoef, f, k, trg + 3 * p0,
                x0 + 3 * p0, pts + 9 * p0, ell + 4 * p0, jump + p0, r0patch + p0,
                r0coef + 16 * p0, mu, work, W + p0 * 9 * Nc, stream);
            if (rc) return rc;
        }
        return SF_OK;
    }
    SurfArgs A;
    A.cnodes = cnodes; A.cnrm = cnrm; A.cw = cw; A.nt = nt; A.nph = nph;
    A.fnodes = fnodes; A.fnrm = fnrm; A.fw = fw; A.fcoef = fcoef; A.f = f;
    A.npairs = npairs; A.trg = trg; A.x0 = x0; A.pts = pts; A.ell = ell; A.jump = jump;
    A.r0patch = r0patch; A.r0coef = r0coef; A.pref = -3.0 / (4.0 * M_PI * mu);
    A.rs = work;
    A.rs_part = work + 9 * npairs;
    A.W = W;
    const int64_t nfine = nt * nph * f * f * 16;
    surf_rs_partial<<<dim3(kSurfRsBlocks, (unsigned)npairs), kSurfThreads, 0, st>>>(A, nfine);
    int rc = check_launch("surf_rs_partial");
    if (rc) return rc;
    surf_rs_final<<<(unsigned)npairs, 32, 0, st>>>(A);
    rc = check_launch("surf_rs_final");
    if (rc) return rc;
    const size_t smem = sizeof(double) * 17 * (size_t)f * f * 16;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(surf_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    surf_patch_kernel<<<dim3((unsigned)(nt * nph), (unsigned)npairs), kSurfThreads, smem, st>>>(A);
    return check_launch("surf_patch_kernel");
}
