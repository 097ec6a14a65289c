// sf_cross.cu — fiber <-> surface interactions evaluated once per pair.
//
// complementary_velocities (system.py:655-687) sums, over every (fiber
// point i, surface node j) pair, two kernels that share the pair geometry:
//   fiber target  i  <- surface source j : stresslet  (q_j w_j . r)(n_j . r) r / r^5
//   surface target j <- fiber source  i  : Stokeslet + (eps L)^2/2 doublet of w_i f_i
// with r = x_i - x_j (the doublet/Stokeslet terms are even in r).  Evaluating
// both from one r, r^2, 1/r, 1/r^3, 1/r^5 costs 14 + 11 + 12 = 37 FP64
// instructions per pair instead of 25 + 26 in two separate sweeps.
//
// Layout and determinism follow sf_sym.cu: fiber points are split into GA
// units of MA points, surface nodes into GB units of MB nodes; one CTA per
// (A unit g, B unit h) task writes
//     partA[h][points of g]   (stresslet sums of g's fiber points over h)
//     partB[g][nodes of h]    (SBT sums of h's surface nodes over g)
// and an ordered pass sums the slots.  Inside a task, the 4 warps hold the
// same 32*TBI fiber points in registers (TBI per lane) and split the
// surface slabs (32 nodes, staged in shared memory); within a slab the 32
// surface accumulators rotate around the warp by shuffles.
#include <cstdlib>
#include <type_traits>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {
namespace {

constexpr int kCrossThreads = 128;

struct __align__(16) CrossA {   // fiber point: x, w f, c = (eps L)^2/2, 3c
    double x, y, z, fx, fy, fz, c, c3;
};
struct __align__(16) CrossB {   // surface node: x, w q, n, pad
    double x, y, z, qx, qy, qz, nx, ny, nz, pad;
};
struct __align__(16) CrossBox {  // bounding box of a 32-point slab
    double lo[3], hi[3];
};

struct CrossArgs {
    const CrossA *a;
    const CrossB *b;
    const CrossBox *abox, *bbox;
    int64_t NA, NB;
    int MA, MB, GA, GB;
    double *partA;               // (GB, NA, 3)
    double *partB;               // (GA, NB, 3)
    unsigned long long *bad_a, *bad_b;
};

__global__ void cross_pack_a(const double *__restrict__ x, const double *__restrict__ f,
                             const double *__restrict__ w, const double *__restrict__ dcoef,
                             int64_t n, CrossA *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double wj = w ? w[j] : 1.0, c = dcoef ? dcoef[j] : 0.0;
        CrossA p;
        p.x = x[3 * j]; p.y = x[3 * j + 1]; p.z = x[3 * j + 2];
        p.fx = wj * f[3 * j]; p.fy = wj * f[3 * j + 1]; p.fz = wj * f[3 * j + 2];
        p.c = c; p.c3 = 3.0 * c;
        out[j] = p;
    }
}

__global__ void cross_pack_b(const double *__restrict__ x, const double *__restrict__ q,
                             const double *__restrict__ w, const double *__restrict__ nrm,
                             int64_t n, CrossB *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double wj = w[j];
        CrossB p;
        p.x = x[3 * j]; p.y = x[3 * j + 1]; p.z = x[3 * j + 2];
        p.qx = wj * q[3 * j]; p.qy = wj * q[3 * j + 1]; p.qz = wj * q[3 * j + 2];
        p.nx = nrm[3 * j]; p.ny = nrm[3 * j + 1]; p.nz = nrm[3 * j + 2];
        p.pad = 0.0;
        out[j] = p;
    }
}

// Slab bounding boxes (warp per slab) of a packed array with x,y,z first.
template <class T>
__global__ void cross_box_kernel(const T *__restrict__ src, int64_t n, CrossBox *__restrict__ box) {
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s * 32 >= n) return;
    const int64_t j = s * 32 + lane;
    double v[6];
    if (j < n) {
        v[0] = v[3] = src[j].x; v[1] = v[4] = src[j].y; v[2] = v[5] = src[j].z;
    } else {
        v[0] = v[1] = v[2] = 1e300;
        v[3] = v[4] = v[5] = -1e300;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            v[c] = fmin(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
            v[3 + c] = fmax(v[3 + c], __shfl_xor_sync(0xffffffffu, v[3 + c], o));
        }
    if (lane == 0) {
        CrossBox b;
        for (int c = 0; c < 3; ++c) { b.lo[c] = v[c]; b.hi[c] = v[3 + c]; }
        box[s] = b;
    }
}

__device__ __forceinline__ bool cross_far(const double *lo, const double *hi, const CrossBox &m) {
    double d2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double gap = fmax(0.0, fmax(m.lo[c] - hi[c], lo[c] - m.hi[c]));
        d2 = fma(gap, gap, d2);
    }
    return d2 > 1e-20;
}

// One (fiber i, surface j) pair, both directions.
template <bool CHECK>
__device__ __forceinline__ void cross_pair(const CrossA &pi, const CrossB &pj, double *ui,
                                           double *uj, int &nb) {
    const double rx = pi.x - pj.x, ry = pi.y - pj.y, rz = pi.z - pj.z;
    const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
    double y0 = rsq_seed(r2);
    if (CHECK) {
        const bool small = below_min_sep(r2);
        nb += small ? 1 : 0;
        y0 = small ? 0.0 : y0;
    }
    const double ir = rsq_refine(r2, y0);
    const double ir2 = ir * ir;
    const double ir3 = ir * ir2;
    const double ir5 = ir3 * ir2;
    {   // fiber target <- surface source: stresslet (pref applied in the reduce)
        const double qr = fma(rz, pj.qz, fma(ry, pj.qy, rx * pj.qx));
        const double nr = fma(rz, pj.nz, fma(ry, pj.ny, rx * pj.nx));
        const double s = qr * nr;
        const double s5 = s * ir5;
        ui[0] = fma(s5, rx, ui[0]);
        ui[1] = fma(s5, ry, ui[1]);
        ui[2] = fma(s5, rz, ui[2]);
    }
    {   // surface target <- fiber source: Stokeslet + doublet, even in r
        const double a = fma(pi.c, ir3, ir);
        const double bb = fma(-pi.c3, ir5, ir3);
        const double rf = fma(rz, pi.fz, fma(ry, pi.fy, rx * pi.fx));
        const double b = rf * bb;
        uj[0] = fma(a, pi.fx, uj[0]);
        uj[1] = fma(a, pi.fy, uj[1]);
        uj[2] = fma(a, pi.fz, uj[2]);
        uj[0] = fma(b, rx, uj[0]);
        uj[1] = fma(b, ry, uj[1]);
        uj[2] = fma(b, rz, uj[2]);
    }
}

template <int TBI>
__global__ void __launch_bounds__(kCrossThreads, 2) cross_task_kernel(CrossArgs A) {
    constexpr int kI = 32 * TBI;
    extern __shared__ double jacc_s[];                     // MB x 3 surface accumulators
    __shared__ double ui_s[4][kI][3];
    __shared__ double2 js_xy[4][32], js_zq[4][32], js_qq[4][32], js_nn[4][32];
    __shared__ double js_nz[4][32];
    const int64_t t = blockIdx.x;
    const int g = (int)(t / A.GB), h = (int)(t - (int64_t)g * A.GB);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t)g * A.MA, h0 = (int64_t)h * A.MB;
    const int ng = (int)min((int64_t)A.MA, A.NA - g0), nh = (int)min((int64_t)A.MB, A.NB - h0);
    const int nslab = (nh + 31) / 32;
    for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x) jacc_s[e] = 0.0;
    __syncthreads();   // zero-fill (any warp) before the owning warp's first +=
    int nb_a = 0, nb_b = 0;
    for (int ib = 0; ib < ng; ib += kI) {
        CrossA pi[TBI];
        double ui[TBI][3];
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            const int il = ib + 32 * k + lane;
            if (il < ng) {
                pi[k] = A.a[g0 + il];
            } else {   // far away and strengthless: contributes exactly 0 both ways
                pi[k].x = pi[k].y = pi[k].z = 1e30;
                pi[k].fx = pi[k].fy = pi[k].fz = pi[k].c = pi[k].c3 = 0.0;
            }
            ui[k][0] = ui[k][1] = ui[k][2] = 0.0;
        }
        double blo[3], bhi[3];
        {
            const CrossBox &m0 = A.abox[(g0 + ib) / 32];
            for (int c = 0; c < 3; ++c) { blo[c] = m0.lo[c]; bhi[c] = m0.hi[c]; }
            for (int k = 1; k < TBI; ++k) {
                if (ib + 32 * k >= ng) break;
                const CrossBox &m1 = A.abox[(g0 + ib) / 32 + k];
                for (int c = 0; c < 3; ++c) {
                    blo[c] = fmin(blo[c], m1.lo[c]);
                    bhi[c] = fmax(bhi[c], m1.hi[c]);
                }
            }
        }
        for (int sl = warp; sl < nslab; sl += 4) {
            const int jl = sl * 32 + lane;
            {
                CrossB q;
                if (jl < nh) {
                    q = A.b[h0 + jl];
                } else {
                    q.x = q.y = q.z = -1e30;
                    q.qx = q.qy = q.qz = q.nx = q.ny = q.nz = 0.0;
                }
                js_xy[warp][lane] = make_double2(q.x, q.y);
                js_zq[warp][lane] = make_double2(q.z, q.qx);
                js_qq[warp][lane] = make_double2(q.qy, q.qz);
                js_nn[warp][lane] = make_double2(q.nx, q.ny);
                js_nz[warp][lane] = q.nz;
            }
            __syncwarp();
            double uj[3] = {0, 0, 0};
            const bool fast = cross_far(blo, bhi, A.bbox[h0 / 32 + sl]);
            const int nxt = (lane + 1) & 31;
            auto step = [&](int s, auto check) {
                const int k = (lane + s) & 31;
                CrossB pj;
                const double2 xy = js_xy[warp][k], zq = js_zq[warp][k], qq = js_qq[warp][k],
                              nn = js_nn[warp][k];
                pj.x = xy.x; pj.y = xy.y; pj.z = zq.x; pj.qx = zq.y; pj.qy = qq.x; pj.qz = qq.y;
                pj.nx = nn.x; pj.ny = nn.y; pj.nz = js_nz[warp][k];
                int nbs = 0;
#pragma unroll
                for (int q = 0; q < TBI; ++q) cross_pair<decltype(check)::value>(pi[q], pj, ui[q], uj, nbs);
                if (decltype(check)::value) {   // padding points sit at +-1e30: never small
                    nb_a += nbs;
                    nb_b += nbs;
                }
                uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
            };
            if (fast) {
#pragma unroll 4
                for (int s = 0; s < 32; ++s) step(s, std::false_type{});
            } else {
                for (int s = 0; s < 32; ++s) step(s, std::true_type{});
            }
            __syncwarp();
            if (jl < nh) {
                double *dst = jacc_s + 3 * jl;
                dst[0] += uj[0];
                dst[1] += uj[1];
                dst[2] += uj[2];
            }
        }
        // combine the 4 warps' fiber partials in warp order, write slot h
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
                __stcs(&A.partA[((int64_t)h * A.NA + g0 + ib + il) * 3 + c], s);
            }
        }
        __syncthreads();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x)
        __stcs(&A.partB[((int64_t)g * A.NB + h0) * 3 + e], jacc_s[e]);
    if (A.bad_a) {
        nb_a = warp_sum_int(nb_a);
        nb_b = warp_sum_int(nb_b);
        if (lane == 0 && nb_a) atomicAdd(A.bad_a, (unsigned long long)nb_a);
        if (lane == 0 && nb_b) atomicAdd(A.bad_b, (unsigned long long)nb_b);
    }
}

// out[i] (+)= pref * sum_s part[s][i], slots in order.
__global__ void cross_reduce_kernel(const double *__restrict__ part, int G, int64_t N,
                                    double pref, double *__restrict__ out, int accumulate) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 3 * N) return;
    double s = 0.0;
    for (int k = 0; k < G; ++k) s += part[(int64_t)k * 3 * N + e];
    out[e] = accumulate ? out[e] + pref * s : pref * s;
}

int round_to(int64_t v, int64_t m) { return (int)((v + m - 1) / m * m); }

}  // namespace

bool use_cross(int64_t NA, int64_t NB) {
    const char *e = getenv("SF_CROSS");
    if (e && atoi(e) == 0) return false;
    if (e && atoi(e) == 2) return NA > 0 && NB > 0;   // forced on (A/B measurements)
    // small surfaces (a C2 particle, 1,024 nodes) give tasks too short to
    // beat the two tiled sweeps; the C4 periphery (40,960 nodes) gains 7 %
    return NA >= 4096 && NB >= 4096;
}

// Unit sizes: MB a multiple of the 32-node slab, MA of the 128-point
// i-sub-block, chosen so the GA x GB tasks fill the GPU (>= ~2048 tasks).
void cross_units(int64_t NA, int64_t NB, int *MA, int *MB) {
    int64_t mb = (NB + 15) / 16;
    mb = mb < 32 ? 32 : (mb > 2048 ? 2048 : mb);
    mb = round_to(mb, 32);
    const int64_t GB = (NB + mb - 1) / mb;
    const int64_t want_ga = (2048 + GB - 1) / GB;
    int64_t ma = NA / want_ga;
    ma = (ma / 128) * 128;
    ma = ma < 128 ? 128 : (ma > 2048 ? 2048 : ma);
    *MA = (int)ma;
    *MB = (int)mb;
}

int pairs_cross(const double *xa, const double *fa, const double *wa, const double *dcoef,
                int64_t NA, const double *xb, const double *qb, const double *wb,
                const double *nb, int64_t NB, double pref_a, double pref_b, double *out_a,
                int accumulate_a, double *out_b, int accumulate_b, int64_t *bad_a,
                int64_t *bad_b, cudaStream_t st, Workspace &ws) {
    if (NA == 0 || NB == 0) return SF_OK;
    int MA, MB;
    cross_units(NA, NB, &MA, &MB);
    const int GA = (int)((NA + MA - 1) / MA), GB = (int)((NB + MB - 1) / MB);
    // workspace slots 7..10 (the pair engine and sf_sym use 0..6)
    CrossA *pa = (CrossA *)ws.get(7, sizeof(CrossA) * (size_t)NA, st);
    CrossB *pb = (CrossB *)ws.get(8, sizeof(CrossB) * (size_t)NB, st);
    const int64_t sa = (NA + 31) / 32, sb = (NB + 31) / 32;
    CrossBox *boxes = (CrossBox *)ws.get(9, sizeof(CrossBox) * (size_t)(sa + sb), st);
    double *part = (double *)ws.get(10, sizeof(double) * 3 * ((size_t)GB * NA + (size_t)GA * NB), st);
    if (!pa || !pb || !boxes || !part) return SF_ENOMEM;
    auto grid = [](int64_t n) { int64_t g = (n + 255) / 256; return (unsigned)(g > 4096 ? 4096 : g); };
    cross_pack_a<<<grid(NA), 256, 0, st>>>(xa, fa, wa, dcoef, NA, pa);
    cross_pack_b<<<grid(NB), 256, 0, st>>>(xb, qb, wb, nb, NB, pb);
    cross_box_kernel<CrossA><<<(unsigned)((sa + 7) / 8), 256, 0, st>>>(pa, NA, boxes);
    cross_box_kernel<CrossB><<<(unsigned)((sb + 7) / 8), 256, 0, st>>>(pb, NB, boxes + sa);
    int rc = check_launch("cross pack");
    if (rc) return rc;
    CrossArgs a;
    a.a = pa; a.b = pb; a.abox = boxes; a.bbox = boxes + sa;
    a.NA = NA; a.NB = NB; a.MA = MA; a.MB = MB; a.GA = GA; a.GB = GB;
    a.partA = part;
    a.partB = part + 3 * (size_t)GB * NA;
    a.bad_a = (unsigned long long *)bad_a;
    a.bad_b = (unsigned long long *)bad_b;
    const size_t smem = sizeof(double) * 3 * (size_t)MB;
    if (cudaFuncSetAttribute(cross_task_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("cudaFuncSetAttribute");
    cross_task_kernel<4><<<(unsigned)((int64_t)GA * GB), kCrossThreads, smem, st>>>(a);
    rc = check_launch("cross_task_kernel");
    if (rc) return rc;
    cross_reduce_kernel<<<(unsigned)((3 * NA + 255) / 256), 256, 0, st>>>(a.partA, GB, NA, pref_a,
                                                                         out_a, accumulate_a);
    cross_reduce_kernel<<<(unsigned)((3 * NB + 255) / 256), 256, 0, st>>>(a.partB, GA, NB, pref_b,
                                                                         out_b, accumulate_b);
    return check_launch("cross_reduce_kernel");
}

}  // namespace sf
