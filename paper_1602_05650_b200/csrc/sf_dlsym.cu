// sf_dlsym.cu — symmetric evaluation of the on-surface subtracted double
// layer (kernels.py:216-249, body.py:254-262) for large meshes.
//
// For nodes i != j with r = x_i - x_j and dq = q_j - q_i the two directed
// terms share r, 1/r^5 and (dq . r):
//   u_i += (w_j n_j . r) (dq . r) r / r^5
//   u_j += (w_i n_i . r) (dq . r) r / r^5      (r -> -r, dq -> -dq)
// so one geometry serves both: 21 shared + 2 x 7 FP64 instructions per
// unordered pair instead of 2 x 24.  Tasks, slots and the ordered reduce
// follow sf_sym.cu (unit pairs {g <= h}; diagonal tasks evaluate the owner
// direction only; j == i is excluded by index as in the reference).
#include <cstdlib>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {
namespace {

constexpr int kDlThreads = 128;

struct __align__(16) DlNode {   // x, q, w n, global index
    double x, y, z, qx, qy, qz, nx, ny, nz;
    int64_t idx;
};

struct DlArgs {
    const DlNode *p;
    int64_t N;
    int M, G;
    int64_t task0;  // first task of this launch (a rank's share)
    double *part;   // (G, N, 3)
};

__global__ void dl_pack(const double *__restrict__ x, const double *__restrict__ nrm,
                        const double *__restrict__ w, const double *__restrict__ q, int64_t n,
                        DlNode *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        DlNode p;
        p.x = x[3 * j]; p.y = x[3 * j + 1]; p.z = x[3 * j + 2];
        p.qx = q[3 * j]; p.qy = q[3 * j + 1]; p.qz = q[3 * j + 2];
        p.nx = w[j] * nrm[3 * j]; p.ny = w[j] * nrm[3 * j + 1]; p.nz = w[j] * nrm[3 * j + 2];
        p.idx = j;
        out[j] = p;
    }
}

template <bool BOTH>
__device__ __forceinline__ void dl_pair(const DlNode &pi, const DlNode &pj, double *ui,
                                        double *uj) {
    const double rx = pi.x - pj.x, ry = pi.y - pj.y, rz = pi.z - pj.z;
    const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
    const double y0 = pi.idx == pj.idx ? 0.0 : rsq_seed(r2);    // j == i excluded
    const double ir = rsq_refine(r2, y0);
    const double ir2 = ir * ir;
    const double ir5 = ir * ir2 * ir2;
    const double dqx = pj.qx - pi.qx, dqy = pj.qy - pi.qy, dqz = pj.qz - pi.qz;
    const double qr5 = fma(dqx, rx, fma(dqy, ry, dqz * rz)) * ir5;
    {
        const double c = fma(pj.nx, rx, fma(pj.ny, ry, pj.nz * rz)) * qr5;
        ui[0] = fma(c, rx, ui[0]);
        ui[1] = fma(c, ry, ui[1]);
        ui[2] = fma(c, rz, ui[2]);
    }
    if (BOTH) {
        const double c = fma(pi.nx, rx, fma(pi.ny, ry, pi.nz * rz)) * qr5;
        uj[0] = fma(c, rx, uj[0]);
        uj[1] = fma(c, ry, uj[1]);
        uj[2] = fma(c, rz, uj[2]);
    }
}

// The TBI pairs of one step, phase by phase (shared j operands in one slot).
template <int TBI>
__device__ __forceinline__ void dl_step_grouped(const DlNode (&pi)[TBI], const DlNode &pj,
                                                double (&ui)[TBI][3], double *uj) {
    double rx[TBI], ry[TBI], rz[TBI], qr5[TBI];
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        rx[q] = pi[q].x - pj.x;
        ry[q] = pi[q].y - pj.y;
        rz[q] = pi[q].z - pj.z;
    }
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        const double r2 = fma(rx[q], rx[q], fma(ry[q], ry[q], rz[q] * rz[q]));
        const double ir = rsq_refine(r2, rsq_seed(r2));
        const double ir2 = ir * ir;
        const double dqx = pj.qx - pi[q].qx, dqy = pj.qy - pi[q].qy, dqz = pj.qz - pi[q].qz;
        qr5[q] = fma(dqx, rx[q], fma(dqy, ry[q], dqz * rz[q])) * (ir * ir2 * ir2);
    }
    double c[TBI];
#pragma unroll
    for (int q = 0; q < TBI; ++q) c[q] = rx[q] * pj.nx;
#pragma unroll
    for (int q = 0; q < TBI; ++q) c[q] = fma(ry[q], pj.ny, c[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) c[q] = fma(rz[q], pj.nz, c[q]) * qr5[q];
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        ui[q][0] = fma(c[q], rx[q], ui[q][0]);
        ui[q][1] = fma(c[q], ry[q], ui[q][1]);
        ui[q][2] = fma(c[q], rz[q], ui[q][2]);
    }
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        const double cj = fma(pi[q].nx, rx[q], fma(pi[q].ny, ry[q], pi[q].nz * rz[q])) * qr5[q];
        uj[0] = fma(cj, rx[q], uj[0]);
        uj[1] = fma(cj, ry[q], uj[1]);
        uj[2] = fma(cj, rz[q], uj[2]);
    }
}

__device__ __forceinline__ void dl_task_units(int64_t t, int G, int &g, int &h) {
    double Gd = (double)G;
    double disc = (2.0 * Gd + 1.0) * (2.0 * Gd + 1.0) - 8.0 * (double)t;
    int r = (int)floor(((2.0 * Gd + 1.0) - sqrt(disc)) * 0.5);
    if (r < 0) r = 0;
    auto start = [&](int row) { return (int64_t)row * G - (int64_t)row * (row - 1) / 2; };
    while (r > 0 && start(r) > t) --r;
    while (r + 1 < G && start(r + 1) <= t) ++r;
    g = r;
    h = r + (int)(t - start(r));
}

template <int TBI, bool GRP>
__global__ void __launch_bounds__(kDlThreads, 2) dl_task_kernel(DlArgs A) {
    constexpr int kI = 32 * TBI;
    extern __shared__ double jacc_s[];
    __shared__ double ui_s[4][kI][3];
    __shared__ DlNode js[4][32];
    int g, h;
    dl_task_units(A.task0 + blockIdx.x, A.G, g, h);
    const bool both = g != h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t)g * A.M, h0 = (int64_t)h * A.M;
    const int ng = (int)min((int64_t)A.M, A.N - g0), nh = (int)min((int64_t)A.M, A.N - h0);
    const int nslab = (nh + 31) / 32;
    if (both)
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x) jacc_s[e] = 0.0;
    __syncthreads();   // zero-fill (any warp) before the owning warp's first +=
    for (int ib = 0; ib < ng; ib += kI) {
        DlNode pi[TBI];
        double ui[TBI][3];
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            const int il = ib + 32 * k + lane;
            if (il < ng) {
                pi[k] = A.p[g0 + il];
            } else {   // far away, zero density and normal: contributes 0 both ways
                pi[k].x = pi[k].y = pi[k].z = 1e30;
                pi[k].qx = pi[k].qy = pi[k].qz = pi[k].nx = pi[k].ny = pi[k].nz = 0.0;
                pi[k].idx = -1;
            }
            ui[k][0] = ui[k][1] = ui[k][2] = 0.0;
        }
        for (int sl = warp; sl < nslab; sl += 4) {
            const int jl = sl * 32 + lane;
            if (jl < nh) {
                js[warp][lane] = A.p[h0 + jl];
            } else {
                DlNode q;
                q.x = q.y = q.z = -1e30;
                q.qx = q.qy = q.qz = q.nx = q.ny = q.nz = 0.0;
                q.idx = -2;
                js[warp][lane] = q;
            }
            __syncwarp();
            double uj[3] = {0, 0, 0};
            const int nxt = (lane + 1) & 31;
            if (both) {
#pragma unroll 2
                for (int s = 0; s < 32; ++s) {
                    const DlNode pj = js[warp][(lane + s) & 31];
                    if (GRP) {
                        dl_step_grouped<TBI>(pi, pj, ui, uj);
                    } else {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) dl_pair<true>(pi[q], pj, ui[q], uj);
                    }
                    uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                    uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                    uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                }
            } else {
#pragma unroll 2
                for (int s = 0; s < 32; ++s) {
                    const DlNode pj = js[warp][(lane + s) & 31];
#pragma unroll
                    for (int q = 0; q < TBI; ++q) dl_pair<false>(pi[q], pj, ui[q], uj);
                }
            }
            __syncwarp();
            if (both && jl < nh) {
                double *dst = jacc_s + 3 * jl;
                dst[0] += uj[0];
                dst[1] += uj[1];
                dst[2] += uj[2];
            }
        }
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            ui_s[warp][32 * k + lane][0] = ui[k][0];
            ui_s[warp][32 * k + lane][1] = ui[k][1];
            ui_s[warp][32 * k + lane][2] = ui[k][2];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * kI; e += blockDim.x) {
            const int il = e / 3, c = e - 3 * il;
            if (ib + il < ng) {
                const double s = ((ui_s[0][il][c] + ui_s[1][il][c]) + ui_s[2][il][c]) + ui_s[3][il][c];
                __stcs(&A.part[((int64_t)h * A.N + g0 + ib + il) * 3 + c], s);
            }
        }
        __syncthreads();
    }
    if (both) {
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x)
            __stcs(&A.part[((int64_t)g * A.N + h0) * 3 + e], jacc_s[e]);
    }
}

// Slot k of a point in unit u was written by task {min(u,k), max(u,k)};
// slots of tasks outside [t0, t1) (another rank's share) are skipped.
__global__ void dl_reduce_kernel(const double *__restrict__ part, int G, int64_t N, int M,
                                 int64_t t0, int64_t t1, double pref, double *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 3 * N) return;
    const int64_t u = (e / 3) / M;
    double s = 0.0;
    for (int k = 0; k < G; ++k) {
        const int64_t g = k < u ? k : u, h = k < u ? u : k;
        const int64_t t = g * G - g * (g - 1) / 2 + (h - g);
        if (t < t0 || t >= t1) continue;
        s += part[(int64_t)k * 3 * N + e];
    }
    out[e] = pref * s;
}

}  // namespace

bool use_dl_symmetric(int64_t n) {
    const char *e = getenv("SF_SYMMETRIC");
    if (e && atoi(e) == 0) return false;
    return n >= 8192;
}

int pairs_dl_subtracted_symmetric(const double *nodes, const double *nrm, const double *w,
                                  const double *q, int64_t n, double pref, double *out,
                                  cudaStream_t st, Workspace &ws, int rank, int world) {
    if (n == 0) return SF_OK;
    int64_t M = n / 128;   // >= 8256 unit-pair tasks, as sym_unit_size
    // (tasks split by cost over ranks as in sf_sym.cu: sym_task_range)
    M = M < 256 ? 256 : (M > 2048 ? 2048 : M);
    M = (M / 128) * 128;
    const int G = (int)((n + M - 1) / M);
    DlNode *packed = (DlNode *)ws.get(3, sizeof(DlNode) * (size_t)n, st);
    double *part = (double *)ws.get(5, sizeof(double) * 3 * (size_t)n * G, st);
    if (!packed || !part) return SF_ENOMEM;
    int64_t pg = (n + 255) / 256;
    dl_pack<<<(unsigned)(pg > 4096 ? 4096 : pg), 256, 0, st>>>(nodes, nrm, w, q, n, packed);
    DlArgs a;
    a.p = packed; a.N = n; a.M = (int)M; a.G = G; a.part = part;
    int64_t ntasks = 0;
    a.task0 = sym_task_range(G, n, M, rank, world, &ntasks);
    const size_t smem = sizeof(double) * 3 * (size_t)M;
    static const bool grouped = [] {
        const char *e = getenv("SF_DL_GROUPED");
        return !(e && e[0] == '0');
    }();
    auto kern = grouped ? dl_task_kernel<4, true> : dl_task_kernel<4, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    if (ntasks > 0) kern<<<(unsigned)ntasks, kDlThreads, smem, st>>>(a);
    int rc = check_launch("dl_task_kernel");
    if (rc) return rc;
    dl_reduce_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, st>>>(part, G, n, (int)M, a.task0,
                                                                     a.task0 + ntasks, pref, out);
    return check_launch("dl_reduce_kernel");
}

}  // namespace sf
