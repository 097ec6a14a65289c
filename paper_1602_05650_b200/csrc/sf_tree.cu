// sf_tree.cu — the reference's TreeSummation backend (system.py:108-224) on
// the device: octree Stokeslet summation with monopole + dipole cells.
//
// The host builds the octree TOPOLOGY from the source positions (the
// reference's octant split, system.py:112-140) and permutes the sources so
// every node owns a contiguous range; per call the device computes the node
// moments from the strengths (centroid c, radius s, F = sum f, D = f^T dy,
// A2 = sum |f| |dy|^2, Fabs = sum |f|), then traverses the tree for every
// target with the reference's opening test
//     d > 0  and  s <= theta d  and  C2 A2 <= tol Fabs d^2
// (far cells: monopole + dipole field, system.py:143-154; leaves: direct
// Stokeslet sums skipping r^2 < 1e-24 like kernels.stokeslet_sum), and
// finally subtracts each target's same-group direct partial (group
// exclusion, system.py:189-200).
//
// Traversal is warp-cooperative: a warp carries 32 targets down the tree
// with a per-node lane mask, visiting nodes in the reference's stack order
// (children pushed in octant order, popped last-first); a lane descends
// only where its own test fails, so each target sees exactly the
// reference's far/near decisions.
#include <cmath>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {
namespace {

constexpr int kTreeWarps = 4;
constexpr int kTreeStack = 8 * 49 + 8;

struct TreeNode {          // device-side node moments (per call)
    double c[3], s, F[3], D[9], A2, Fabs;
};

// One warp per node: two passes over the node's contiguous source range.
__global__ void tree_moments_kernel(const double *__restrict__ src, const double *__restrict__ f,
                                    const int64_t *__restrict__ nbeg,
                                    const int64_t *__restrict__ nend, int64_t nnodes,
                                    TreeNode *__restrict__ out) {
    const int64_t node = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (node >= nnodes) return;
    const int64_t b = nbeg[node], e = nend[node];
    const double cnt = (double)(e - b);
    double sx = 0, sy = 0, sz = 0;
    for (int64_t i = b + lane; i < e; i += 32) {
        sx += src[3 * i];
        sy += src[3 * i + 1];
        sz += src[3 * i + 2];
    }
    const double c0 = warp_sum(sx) / cnt, c1 = warp_sum(sy) / cnt, c2 = warp_sum(sz) / cnt;
    double r2max = 0.0, F[3] = {0, 0, 0}, D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, A2 = 0.0, Fa = 0.0;
    for (int64_t i = b + lane; i < e; i += 32) {
        const double dy[3] = {src[3 * i] - c0, src[3 * i + 1] - c1, src[3 * i + 2] - c2};
        const double fi[3] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
        const double r2 = dy[0] * dy[0] + dy[1] * dy[1] + dy[2] * dy[2];
        r2max = fmax(r2max, r2);
        const double fn = sqrt(fi[0] * fi[0] + fi[1] * fi[1] + fi[2] * fi[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            F[a] += fi[a];
#pragma unroll
            for (int c = 0; c < 3; ++c) D[3 * a + c] += fi[a] * dy[c];
        }
        A2 += fn * r2;
        Fa += fn;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2max = fmax(r2max, __shfl_xor_sync(0xffffffffu, r2max, o));
    TreeNode t;
    t.c[0] = c0; t.c[1] = c1; t.c[2] = c2;
    t.s = sqrt(r2max);
#pragma unroll
    for (int a = 0; a < 3; ++a) t.F[a] = warp_sum(F[a]);
#pragma unroll
    for (int a = 0; a < 9; ++a) t.D[a] = warp_sum(D[a]);
    t.A2 = warp_sum(A2);
    t.Fabs = warp_sum(Fa);
    if (lane == 0) out[node] = t;
}

struct TreeArgs {
    const double *trg;          // (nt,3)
    int64_t nt;
    const double *src, *f;      // permuted sources / strengths (ns,3)
    const TreeNode *node;
    const int64_t *nbeg, *nend, *first_child;
    const int *nchild;
    double theta, tol, C2, pref;
    double *out;                // (nt,3)
};

__device__ __forceinline__ void mono_dipole(const double r[3], double d, const TreeNode &n,
                                            double pref, double u[3]) {
    const double id3 = 1.0 / (d * d * d);
    const double rf = r[0] * n.F[0] + r[1] * n.F[1] + r[2] * n.F[2];
    double v[3], Dr[3], DTr[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        Dr[a] = n.D[3 * a] * r[0] + n.D[3 * a + 1] * r[1] + n.D[3 * a + 2] * r[2];
        DTr[a] = n.D[a] * r[0] + n.D[3 + a] * r[1] + n.D[6 + a] * r[2];
    }
    const double rDr = r[0] * Dr[0] + r[1] * Dr[1] + r[2] * Dr[2];
    const double tr = n.D[0] + n.D[4] + n.D[8];
    const double d5 = d * d * d * d * d;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        v[a] = n.F[a] / d + rf * id3 * r[a];
        v[a] += (Dr[a] - DTr[a] - tr * r[a]) * id3;
        v[a] += 3.0 * (rDr / d5) * r[a];
        u[a] += pref * v[a];
    }
}

__global__ void __launch_bounds__(32 * kTreeWarps) tree_eval_kernel(TreeArgs A) {
    __shared__ int64_t st_node[kTreeWarps][kTreeStack];
    __shared__ unsigned st_mask[kTreeWarps][kTreeStack];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = ((int64_t)blockIdx.x * kTreeWarps + w) * 32 + lane;
    const bool live = t < A.nt;
    double x[3] = {0, 0, 0}, u[3] = {0, 0, 0};
    if (live) { x[0] = A.trg[3 * t]; x[1] = A.trg[3 * t + 1]; x[2] = A.trg[3 * t + 2]; }
    const unsigned all = __ballot_sync(0xffffffffu, live);
    if (!all) return;
    int sp = 0;
    if (lane == 0) { st_node[w][0] = 0; st_mask[w][0] = all; }
    sp = 1;
    __syncwarp();
    while (sp > 0) {
        --sp;
        const int64_t nd = st_node[w][sp];
        const unsigned mask = st_mask[w][sp];
        __syncwarp();
        const bool act = (mask >> lane) & 1u;
        const int nc = A.nchild[nd];
        if (nc == 0) {   // leaf: direct sum over its sources (kernels.stokeslet_sum)
            if (act) {
                const int64_t b = A.nbeg[nd], e = A.nend[nd];
                for (int64_t j = b; j < e; ++j) {
                    const double r0 = x[0] - A.src[3 * j], r1 = x[1] - A.src[3 * j + 1],
                                 r2 = x[2] - A.src[3 * j + 2];
                    const double d2 = r0 * r0 + r1 * r1 + r2 * r2;
                    if (d2 < 1e-24) continue;
                    const double d = sqrt(d2);
                    const double f0 = A.f[3 * j], f1 = A.f[3 * j + 1], f2 = A.f[3 * j + 2];
                    const double rf = r0 * f0 + r1 * f1 + r2 * f2;
                    const double id = 1.0 / d, id3 = 1.0 / (d2 * d);
                    u[0] += A.pref * (f0 * id + rf * r0 * id3);
                    u[1] += A.pref * (f1 * id + rf * r1 * id3);
                    u[2] += A.pref * (f2 * id + rf * r2 * id3);
                }
            }
            continue;
        }
        bool open = false;
        if (act) {
            const TreeNode &n = A.node[nd];
            const double r[3] = {x[0] - n.c[0], x[1] - n.c[1], x[2] - n.c[2]};
            const double d = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
            const bool ok = (d > 0.0) && (n.s <= A.theta * d) &&
                            (A.C2 * n.A2 <= A.tol * n.Fabs * d * d);
            if (ok) mono_dipole(r, d, n, A.pref, u);
            open = !ok;
        }
        const unsigned rest = __ballot_sync(0xffffffffu, open);
        if (rest) {
            const int64_t fc = A.first_child[nd];
            if (lane == 0)
                for (int k = 0; k < nc; ++k) {
                    st_node[w][sp + k] = fc + k;
                    st_mask[w][sp + k] = rest;
                }
            sp += nc;
            __syncwarp();
        }
    }
    if (live) {
        A.out[3 * t] = u[0];
        A.out[3 * t + 1] = u[1];
        A.out[3 * t + 2] = u[2];
    }
}

// out[t] -= same-group direct partial: sources of the target's group are
// the contiguous range [gbeg[g], gend[g]) of the group-sorted arrays.
__global__ void tree_group_sub_kernel(const double *__restrict__ trg,
                                      const int64_t *__restrict__ tgrp, int64_t nt,
                                      const double *__restrict__ gsrc,
                                      const double *__restrict__ gf,
                                      const int64_t *__restrict__ gbeg,
                                      const int64_t *__restrict__ gend, int64_t ngroups,
                                      double pref, double *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t g = tgrp[t];
    if (g < 0 || g >= ngroups) return;
    const double x0 = trg[3 * t], x1 = trg[3 * t + 1], x2 = trg[3 * t + 2];
    double u0 = 0, u1 = 0, u2 = 0;
    for (int64_t j = gbeg[g]; j < gend[g]; ++j) {
        const double r0 = x0 - gsrc[3 * j], r1 = x1 - gsrc[3 * j + 1], r2 = x2 - gsrc[3 * j + 2];
        const double d2 = r0 * r0 + r1 * r1 + r2 * r2;
        if (d2 < 1e-24) continue;
        const double d = sqrt(d2);
        const double f0 = gf[3 * j], f1 = gf[3 * j + 1], f2 = gf[3 * j + 2];
        const double rf = r0 * f0 + r1 * f1 + r2 * f2;
        const double id = 1.0 / d, id3 = 1.0 / (d2 * d);
        u0 += pref * (f0 * id + rf * r0 * id3);
        u1 += pref * (f1 * id + rf * r1 * id3);
        u2 += pref * (f2 * id + rf * r2 * id3);
    }
    out[3 * t] -= u0;
    out[3 * t + 1] -= u1;
    out[3 * t + 2] -= u2;
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" int sf_tree_stokeslet(const double *trg, const int64_t *tgrp, int64_t nt,
                                 const double *src, const double *f, int64_t ns,
                                 const int64_t *nbeg, const int64_t *nend,
                                 const int64_t *first_child, const int *nchild, int64_t nnodes,
                                 const double *gsrc, const double *gf, const int64_t *gbeg,
                                 const int64_t *gend, int64_t ngroups, double theta,
                                 double cell_tolerance, double mu, double *work, double *out,
                                 void *stream) {
    if (nt < 0 || ns < 0 || nnodes < 0 || ngroups < 0) return set_error(SF_EINVAL, "negative size");
    if (!(mu > 0)) return set_error(SF_EINVAL, "viscosity must be positive");
    if (nt == 0) return SF_OK;
    if (!trg || !out) return set_error(SF_EINVAL, "null target/output pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const double pref = 1.0 / (8.0 * M_PI * mu);
    if (ns == 0 || nnodes == 0) {
        if (cudaMemsetAsync(out, 0, sizeof(double) * 3 * nt, st) != cudaSuccess)
            return check_launch("memset");
        return SF_OK;
    }
    if (!src || !f || !nbeg || !nend || !first_child || !nchild || !work)
        return set_error(SF_EINVAL, "null tree pointer");
    TreeNode *nodes = reinterpret_cast<TreeNode *>(work);
    tree_moments_kernel<<<(unsigned)((nnodes + 7) / 8), 256, 0, st>>>(src, f, nbeg, nend, nnodes,
                                                                      nodes);
    int rc = check_launch("tree_moments_kernel");
    if (rc) return rc;
    TreeArgs A;
    A.trg = trg; A.nt = nt; A.src = src; A.f = f; A.node = nodes;
    A.nbeg = nbeg; A.nend = nend; A.first_child = first_child; A.nchild = nchild;
    A.theta = theta; A.tol = cell_tolerance; A.C2 = 16.0; A.pref = pref; A.out = out;
    const int64_t warps = (nt + 31) / 32;
    tree_eval_kernel<<<(unsigned)((warps + kTreeWarps - 1) / kTreeWarps), 32 * kTreeWarps, 0,
                       st>>>(A);
    rc = check_launch("tree_eval_kernel");
    if (rc) return rc;
    if (ngroups > 0 && tgrp) {
        if (!gsrc || !gf || !gbeg || !gend) return set_error(SF_EINVAL, "null group pointer");
        tree_group_sub_kernel<<<(unsigned)((nt + 127) / 128), 128, 0, st>>>(
            trg, tgrp, nt, gsrc, gf, gbeg, gend, ngroups, pref, out);
        rc = check_launch("tree_group_sub_kernel");
    }
    return rc;
}

extern "C" int64_t sf_tree_work_doubles(int64_t nnodes) {
    return nnodes * (int64_t)(sizeof(sf::TreeNode) / sizeof(double));
}
