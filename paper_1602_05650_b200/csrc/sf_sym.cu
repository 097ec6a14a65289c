// sf_sym.cu — symmetric evaluation of the fiber-fiber Stokeslet + doublet sum.
//
// When the targets are exactly the sources (the fiber x fiber block of
// complementary_velocities, system.py:656-671), the pair geometry r, r^2,
// 1/r, 1/r^3, 1/r^5 of (i,j) is shared with (j,i): the kernel r_ij r_ij^T /r^3
// is even in r.  Computing both directions from one geometry evaluation costs
// 14 + 2 x 12 = 38 FP64 instructions per unordered pair (19 per pair
// interaction) instead of 2 x 26.
//
// Partial slots are written with streaming stores (st.global.cs): they are
// read once, by the ordered reduce, and must not evict the source records
// that every CTA re-reads from L2.
//
// Determinism without atomics: points are split into G units of M points
// (M a multiple of the fiber size, so units align to fibers).  A task is an
// unordered unit pair {g,h}; the CTA computes every (i in g, j in h) pair in
// both directions and produces two partial sums, the slot-h partial of the
// points of g (sum over j in h, owner direction) and the slot-g partial of
// the points of h (sum over i in g, transposed direction).  Diagonal tasks
// {g,g} produce only the owner direction.  Every point's G partials are
// summed in slot order.  Every partial is produced by one CTA in a fixed
// loop order, so results are bitwise reproducible.
//
// Bounded partial storage: the tasks run in waves, each a contiguous range
// of task rows [ga, gl] (row g = tasks {g, h >= g}).  A wave's partials live
// in a compact buffer: owner partials A[g - ga][h - ga][M points][3] and
// transposed partials B[g - ga][points >= ga M][3]; after the wave, an
// ordered pass adds them to the running per-point sum in slot order.  Along
// one point's slot order the task index increases, so consecutive waves add
// consecutive runs of its slots: the sum is the same sequence of additions
// as one pass over all G slots, bit for bit, for any wave size.  Waves
// alternate over the caller's stream and side streams with one buffer each,
// so one wave's tail overlaps the next wave (SF_SYM_WAVE_MB per buffer,
// SF_SYM_STREAMS buffers/streams).
//
// Inside a task: 4 warps share an i-sub-block of 64 points (2 per lane, in
// registers with their owner accumulators); j runs in 32-point slabs, slab
// k owned by warp k % 4.  Within a slab each lane holds one j (data and
// transposed accumulator) and the 32 j's rotate around the warp with
// shuffles, so every (i, j) of the 64 x 32 block is visited once and each
// j's transposed sum stays in registers; after 32 rotations it is added to
// the task's shared-memory accumulator for that j (always by the same warp,
// in i-sub-block order).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

struct __align__(16) SymSrc {  // same 80-byte record as the pair engine's Src80
    double v[9];
    int g;
    int pad;
};
static_assert(sizeof(SymSrc) == 80, "record must be 80 bytes");

struct __align__(16) SlabMeta {  // bounding box + group range + capsule of 32 points
    double lo[3], hi[3];
    int gmin, gmax;
    // capsule: segment from the slab's first to its last point, radius = the
    // largest point-to-segment distance (a fiber's 32 nodes hug its chord)
    double p0[3], p1[3], rad;
    // the doublet coefficient c shared by the slab's points, NaN when they differ
    // (a fiber-aligned slab has one c: the packed FP32c kernel then takes c_j as
    // a 32-bit broadcast operand instead of a register pair)
    double cuni;
};

struct SymArgs {
    const SymSrc *src;
    const SlabMeta *slab;
    int64_t N;
    int M;
    int G;
    int64_t ntasks;   // tasks of this launch (one wave)
    int64_t task0;    // first task of the wave
    double *partA;    // owner partials (rows, Acols, M, 3) of the wave's rows
    double *partB;    // transposed partials (rows, Bstride, 3)
    int64_t ga;       // first task row of the wave
    int64_t Acols;    // G - ga
    int64_t Bstride;  // N - ga M
    unsigned long long *bad;
    const double *x;  // (N, 3) FP64 positions: the FP32 variant's coincidence test
    int nofast;       // SF_SYM_NOFAST=1: every slab pair on the checked path (cost model)
    int cs;           // partials stored evict-first (waves larger than L2 can keep)
};

// Partial stores: evict-first when the wave's partials would not stay in L2
// anyway (they must not push out the source records, C5), plain write-back
// when they fit and the ordered reduce can read them from L2 (C2: 67 MB).
__device__ __forceinline__ void part_store(const SymArgs &a, double *p, double v) {
    if (a.cs)
        __stcs(p, v);
    else
        *p = v;
}

constexpr int kSymThreads = 128;

// slot-h partial of point g0 + local (owner direction of task {g,h})
__device__ __forceinline__ double *owner_slot(const SymArgs &a, int g, int h, int64_t local) {
    return a.partA + ((((int64_t)g - a.ga) * a.Acols + ((int64_t)h - a.ga)) * a.M + local) * 3;
}
// slot-g partial of point p >= g M (transposed direction of task {g,h})
__device__ __forceinline__ double *trans_slot(const SymArgs &a, int g, int64_t p) {
    return a.partB + ((((int64_t)g - a.ga) * a.Bstride) + (p - a.ga * a.M)) * 3;
}

struct PData {
    double x, y, z, fx, fy, fz, c, c3;
    int g;
};

__device__ __forceinline__ PData load_point(const SymArgs &a, int64_t k, bool valid) {
    PData p;
    if (valid) {
        const double2 *q = reinterpret_cast<const double2 *>(a.src + k);
        const double2 a0 = q[0], a1 = q[1], a2 = q[2], a3 = q[3];
        p.x = a0.x; p.y = a0.y; p.z = a1.x; p.fx = a1.y; p.fy = a2.x; p.fz = a2.y;
        p.c = a3.x; p.c3 = a3.y;
        p.g = a.src[k].g;
    } else {  // far away and strengthless: contributes exactly 0 both ways
        p.x = p.y = p.z = 1e30;
        p.fx = p.fy = p.fz = p.c = p.c3 = 0.0;
        p.g = -3;
    }
    return p;
}

// One unordered pair, both directions.  ui += (j -> i), uj += (i -> j).
template <bool CHECK, bool BOTH>
__device__ __forceinline__ void sym_pair(const PData &pi, const PData &pj, double *ui, double *uj,
                                         int &nb) {
    const double rx = pi.x - pj.x, ry = pi.y - pj.y, rz = pi.z - pj.z;
    const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
    double y0 = rsq_seed(r2);
    if (CHECK) {
        const bool excl = (pi.g == pj.g) && pi.g >= 0;
        const bool small = below_min_sep(r2);
        nb += (small && !excl) ? (BOTH ? 2 : 1) : 0;
        y0 = (excl || small) ? 0.0 : y0;
    }
    const double ir = rsq_refine(r2, y0);
    const double ir2 = ir * ir;
    const double ir3 = ir * ir2;
    const double ir5 = ir3 * ir2;
    {   // j -> i
        const double a = fma(pj.c, ir3, ir);
        const double bb = fma(-pj.c3, ir5, ir3);
        const double rf = fma(rz, pj.fz, fma(ry, pj.fy, rx * pj.fx));
        const double b = rf * bb;
        ui[0] = fma(a, pj.fx, ui[0]);
        ui[1] = fma(a, pj.fy, ui[1]);
        ui[2] = fma(a, pj.fz, ui[2]);
        ui[0] = fma(b, rx, ui[0]);
        ui[1] = fma(b, ry, ui[1]);
        ui[2] = fma(b, rz, ui[2]);
    }
    if (BOTH) {  // i -> j: (r_ji.f) r_ji = (r_ij.f) r_ij
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

// The TBI pairs of one step (fast path, both directions) evaluated phase by
// phase so that consecutive DFMAs share the j operand (c_j, f_j) in one
// slot and can take it from the operand reuse cache: DFMAs with three
// distinct register sources issue at 2/3 rate on sm_100a.
template <int TBI>
__device__ __forceinline__ void sym_step_grouped(const PData (&pi)[TBI], const PData &pj,
                                                 double (&ui)[TBI][3], double *uj) {
    double rx[TBI], ry[TBI], rz[TBI], ir[TBI], ir3[TBI], ir5[TBI];
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        rx[q] = pi[q].x - pj.x;
        ry[q] = pi[q].y - pj.y;
        rz[q] = pi[q].z - pj.z;
    }
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        const double r2 = fma(rx[q], rx[q], fma(ry[q], ry[q], rz[q] * rz[q]));
        ir[q] = rsq_refine(r2, rsq_seed(r2));
        const double ir2 = ir[q] * ir[q];
        ir3[q] = ir[q] * ir2;
        ir5[q] = ir3[q] * ir2;
    }
    double a[TBI], b[TBI];
    // owner direction: coefficients of source j (c_j, 3c_j, f_j shared across q)
#pragma unroll
    for (int q = 0; q < TBI; ++q) a[q] = fma(pj.c, ir3[q], ir[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = rx[q] * pj.fx;
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = fma(ry[q], pj.fy, b[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = fma(rz[q], pj.fz, b[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] *= fma(-pj.c3, ir5[q], ir3[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][0] = fma(a[q], pj.fx, ui[q][0]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][1] = fma(a[q], pj.fy, ui[q][1]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][2] = fma(a[q], pj.fz, ui[q][2]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        ui[q][0] = fma(b[q], rx[q], ui[q][0]);
        ui[q][1] = fma(b[q], ry[q], ui[q][1]);
        ui[q][2] = fma(b[q], rz[q], ui[q][2]);
    }
    // transposed direction: coefficients of the i points
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        const double ai = fma(pi[q].c, ir3[q], ir[q]);
        const double bi = fma(rz[q], pi[q].fz, fma(ry[q], pi[q].fy, rx[q] * pi[q].fx)) *
                          fma(-pi[q].c3, ir5[q], ir3[q]);
        uj[0] = fma(ai, pi[q].fx, uj[0]);
        uj[1] = fma(ai, pi[q].fy, uj[1]);
        uj[2] = fma(ai, pi[q].fz, uj[2]);
        uj[0] = fma(bi, rx[q], uj[0]);
        uj[1] = fma(bi, ry[q], uj[1]);
        uj[2] = fma(bi, rz[q], uj[2]);
    }
}

__device__ __forceinline__ PData shfl_next(const PData &p, int src_lane) {
    PData q;
    q.x = __shfl_sync(0xffffffffu, p.x, src_lane);
    q.y = __shfl_sync(0xffffffffu, p.y, src_lane);
    q.z = __shfl_sync(0xffffffffu, p.z, src_lane);
    q.fx = __shfl_sync(0xffffffffu, p.fx, src_lane);
    q.fy = __shfl_sync(0xffffffffu, p.fy, src_lane);
    q.fz = __shfl_sync(0xffffffffu, p.fz, src_lane);
    q.c = __shfl_sync(0xffffffffu, p.c, src_lane);
    q.c3 = __shfl_sync(0xffffffffu, p.c3, src_lane);
    q.g = __shfl_sync(0xffffffffu, p.g, src_lane);
    return q;
}

__device__ __forceinline__ void task_units(int64_t t, int G, int &g, int &h) {
    // tasks enumerate {g <= h} row by row: row g has G - g entries
    // solve for the row with a float estimate, then fix up
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

__device__ __forceinline__ bool boxes_far(const double *blo, const double *bhi, const SlabMeta &m) {
    double d2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double gap = fmax(0.0, fmax(m.lo[c] - bhi[c], blo[c] - m.hi[c]));
        d2 = fma(gap, gap, d2);
    }
    return d2 > 1e-20;
}

// Squared distance between the segments [p0, p1] and [q0, q1] (closest
// points with the parameters clamped to [0, 1]).
__device__ __forceinline__ double seg_seg_dist2(const double *p0, const double *p1,
                                                const double *q0, const double *q1) {
    double d1[3], d2[3], r[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        d1[c] = p1[c] - p0[c];
        d2[c] = q1[c] - q0[c];
        r[c] = p0[c] - q0[c];
    }
    const double a = d1[0] * d1[0] + d1[1] * d1[1] + d1[2] * d1[2];
    const double e = d2[0] * d2[0] + d2[1] * d2[1] + d2[2] * d2[2];
    const double f = d2[0] * r[0] + d2[1] * r[1] + d2[2] * r[2];
    double sp = 0.0, tq = 0.0;
    if (a > 1e-300 || e > 1e-300) {
        if (a <= 1e-300) {
            tq = fmin(fmax(f / e, 0.0), 1.0);
        } else {
            const double c = d1[0] * r[0] + d1[1] * r[1] + d1[2] * r[2];
            if (e <= 1e-300) {
                sp = fmin(fmax(-c / a, 0.0), 1.0);
            } else {
                const double b = d1[0] * d2[0] + d1[1] * d2[1] + d1[2] * d2[2];
                const double den = a * e - b * b;
                sp = den > 0.0 ? fmin(fmax((b * f - c * e) / den, 0.0), 1.0) : 0.0;
                tq = (b * sp + f) / e;
                if (tq < 0.0) {
                    tq = 0.0;
                    sp = fmin(fmax(-c / a, 0.0), 1.0);
                } else if (tq > 1.0) {
                    tq = 1.0;
                    sp = fmin(fmax((b - c) / a, 0.0), 1.0);
                }
            }
        }
    }
    double d = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double v = (p0[c] + sp * d1[c]) - (q0[c] + tq * d2[c]);
        d = fma(v, v, d);
    }
    return d;
}

// Two slabs' capsules more than 1e-10 apart: every point pair of the two
// slabs is then farther than 1e-10 (the check-free path is exact).  Radial
// aster fibers have overlapping axis-aligned boxes but separate capsules.
__device__ __forceinline__ bool capsules_far(const SlabMeta &a, const SlabMeta &b) {
    if (a.rad < 0.0 || b.rad < 0.0) return false;    // capsules disabled (SF_SYM_CAPSULE=0)
    const double gap = a.rad + b.rad + 1e-10;
    return seg_seg_dist2(a.p0, a.p1, b.p0, b.p1) > gap * gap;
}

// Every i slab of the sub-block (kvalid of them, from global/L1 slab metas)
// farther than 1e-10 from the j slab (boxes, then capsules).  Testing each 32-point slab
// box, rather than the union box of the sub-block, keeps the check-free path
// for asters: fibers fanning out of a centrosome have overlapping union
// boxes for most slab pairs (62 % at C2) but separate slab boxes (97 %).
template <int TBI>
__device__ __forceinline__ bool islabs_far(const SlabMeta *mi, int kvalid, const SlabMeta &mj) {
    bool far = true;
#pragma unroll
    for (int k = 0; k < TBI; ++k) {
        if (k < kvalid) {
            double d2 = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double gap = fmax(0.0, fmax(mj.lo[c] - mi[k].hi[c], mi[k].lo[c] - mj.hi[c]));
                d2 = fma(gap, gap, d2);
            }
            far = far && (d2 > 1e-20 || capsules_far(mi[k], mj));
        }
    }
    return far;
}

template <int MINB, int TBI, bool PF = false, bool GRP = false>
__global__ void __launch_bounds__(kSymThreads, MINB) sym_task_kernel(SymArgs a) {
    constexpr int kI = 32 * TBI;
    extern __shared__ double jacc_s[];           // M x 3 transposed accumulators
    __shared__ double ui_s[4][kI][3];             // per-warp owner partials
    __shared__ double2 js_xy[4][32], js_zf[4][32], js_ff[4][32], js_cc[4][32];  // j slabs
    __shared__ int js_g[4][32];
    if ((int64_t)blockIdx.x >= a.ntasks) return;
    const int64_t t = a.task0 + blockIdx.x;
    int g, h;
    task_units(t, a.G, g, h);
    const bool both = g != h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t)g * a.M, h0 = (int64_t)h * a.M;
    const int ng = (int)min((int64_t)a.M, a.N - g0), nh = (int)min((int64_t)a.M, a.N - h0);
    const int nslab = (nh + 31) / 32;
    if (both)
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x) jacc_s[e] = 0.0;
    __syncthreads();   // zero-fill (any warp) before the owning warp's first +=
    int nb = 0;
    for (int ib = 0; ib < ng; ib += kI) {
        PData pi[TBI];
        double ui[TBI][3];
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            pi[k] = load_point(a, g0 + ib + 32 * k + lane, ib + 32 * k + lane < ng);
            ui[k][0] = ui[k][1] = ui[k][2] = 0.0;
        }
        // union box + group range of this i-sub-block; when the union box
        // touches a j slab, its slab boxes are tested one by one
        const SlabMeta *mi = a.slab + (g0 + ib) / 32;
        const int kvalid = min(TBI, (ng - ib + 31) / 32);
        double blo[3], bhi[3];
        int gmn = mi[0].gmin, gmx = mi[0].gmax;
        for (int c = 0; c < 3; ++c) { blo[c] = mi[0].lo[c]; bhi[c] = mi[0].hi[c]; }
        for (int k = 1; k < kvalid; ++k) {
            for (int c = 0; c < 3; ++c) {
                blo[c] = fmin(blo[c], mi[k].lo[c]);
                bhi[c] = fmax(bhi[c], mi[k].hi[c]);
            }
            gmn = min(gmn, mi[k].gmin);
            gmx = max(gmx, mi[k].gmax);
        }
        for (int sl = warp; sl < nslab; sl += 4) {
            const int jl = sl * 32 + lane;
            {   // stage this warp's slab in shared memory (double2 SoA, conflict-free)
                const PData q = load_point(a, h0 + jl, jl < nh);
                js_xy[warp][lane] = make_double2(q.x, q.y);
                js_zf[warp][lane] = make_double2(q.z, q.fx);
                js_ff[warp][lane] = make_double2(q.fy, q.fz);
                js_cc[warp][lane] = make_double2(q.c, q.c3);
                js_g[warp][lane] = q.g;
            }
            __syncwarp();
            double uj[3] = {0, 0, 0};
            const SlabMeta &mj = a.slab[h0 / 32 + sl];
            const bool fast = !a.nofast && (mj.gmax < gmn || mj.gmin > gmx) &&
                              (boxes_far(blo, bhi, mj) || islabs_far<TBI>(mi, kvalid, mj));
            const int nxt = (lane + 1) & 31;
            // step s: this lane pairs its i's with j = (lane + s) mod 32 and
            // carries that j's transposed accumulator (rotated by shuffles)
            if (both && fast && PF) {
                // positions of step s+1 are loaded while step s computes
                double2 nxy = js_xy[warp][lane], nzf = js_zf[warp][lane];
#pragma unroll 8
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PData pj;
                    const double2 ff = js_ff[warp][k], cc = js_cc[warp][k];
                    pj.x = nxy.x; pj.y = nxy.y; pj.z = nzf.x; pj.fx = nzf.y; pj.fy = ff.x;
                    pj.fz = ff.y; pj.c = cc.x; pj.c3 = cc.y; pj.g = 0;
                    const int k1 = (lane + s + 1) & 31;
                    nxy = js_xy[warp][k1];
                    nzf = js_zf[warp][k1];
                    if (GRP) {
                        sym_step_grouped<TBI>(pi, pj, ui, uj);
                    } else {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) sym_pair<false, true>(pi[q], pj, ui[q], uj, nb);
                    }
                    uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                    uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                    uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                }
            } else if (both && fast) {
#pragma unroll 4
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PData pj;
                    const double2 xy = js_xy[warp][k], zf = js_zf[warp][k], ff = js_ff[warp][k],
                                  cc = js_cc[warp][k];
                    pj.x = xy.x; pj.y = xy.y; pj.z = zf.x; pj.fx = zf.y; pj.fy = ff.x; pj.fz = ff.y;
                    pj.c = cc.x; pj.c3 = cc.y; pj.g = 0;
#pragma unroll
                    for (int q = 0; q < TBI; ++q) sym_pair<false, true>(pi[q], pj, ui[q], uj, nb);
                    uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                    uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                    uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                }
            } else {
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PData pj;
                    const double2 xy = js_xy[warp][k], zf = js_zf[warp][k], ff = js_ff[warp][k],
                                  cc = js_cc[warp][k];
                    pj.x = xy.x; pj.y = xy.y; pj.z = zf.x; pj.fx = zf.y; pj.fy = ff.x; pj.fz = ff.y;
                    pj.c = cc.x; pj.c3 = cc.y; pj.g = js_g[warp][k];
                    int nbi = 0;
                    if (both) {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) sym_pair<true, true>(pi[q], pj, ui[q], uj, nbi);
                        uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                        uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                        uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                    } else if (fast) {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) sym_pair<false, false>(pi[q], pj, ui[q], uj, nbi);
                    } else {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) sym_pair<true, false>(pi[q], pj, ui[q], uj, nbi);
                    }
                    // count only pairs whose both ends are real points
                    if (pj.g != -3) nb += nbi;
                }
            }
            __syncwarp();
            // after 32 rotations each lane again holds its own j's accumulator
            if (both && jl < nh) {
                double *dst = jacc_s + 3 * jl;
                dst[0] += uj[0];
                dst[1] += uj[1];
                dst[2] += uj[2];
            }
        }
        // combine the 4 warps' owner partials in warp order, write slot h
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
                part_store(a, owner_slot(a, g, h, ib + il) + c, s);
            }
        }
        __syncthreads();
    }
    if (both) {
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x)
            part_store(a, trans_slot(a, g, h0) + e, jacc_s[e]);
    }
    // invalid i lanes never count (their g is -3 and they sit at 1e30)
    if (a.bad) {
        nb = warp_sum_int(nb);
        if (lane == 0 && nb) atomicAdd(a.bad, (unsigned long long)nb);
    }
}

// Modelled cost of every unit-pair task (one thread per task), replaying the
// task kernel's slab-pair decisions (TBI = 4 i points per lane): a both-ways
// slab pair on the check-free path costs 1 per (i, j) cell, on the checked
// path c_checked; a diagonal task's cells cost c_diag (one direction at a
// time, always checked).  Cells of invalid lanes count too: the kernel
// evaluates them.  Used to split the tasks over ranks by time, not pairs.
__global__ void sym_task_cost_kernel(const SlabMeta *__restrict__ meta, int64_t N, int M, int G,
                                     int64_t ntasks, double c_checked, double c_diag,
                                     double *__restrict__ cost) {
    constexpr int TBI = 4, kI = 32 * TBI;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntasks) return;
    int g, h;
    task_units(t, G, g, h);
    const bool both = g != h;
    const int64_t g0 = (int64_t)g * M, h0 = (int64_t)h * M;
    const int ng = (int)min((int64_t)M, N - g0), nh = (int)min((int64_t)M, N - h0);
    const int nslab = (nh + 31) / 32;
    double c = 0.0;
    for (int ib = 0; ib < ng; ib += kI) {
        const SlabMeta *mi = meta + (g0 + ib) / 32;
        const int kvalid = min(TBI, (ng - ib + 31) / 32);
        double blo[3], bhi[3];
        int gmn = mi[0].gmin, gmx = mi[0].gmax;
        for (int q = 0; q < 3; ++q) { blo[q] = mi[0].lo[q]; bhi[q] = mi[0].hi[q]; }
        for (int k = 1; k < kvalid; ++k) {
            for (int q = 0; q < 3; ++q) {
                blo[q] = fmin(blo[q], mi[k].lo[q]);
                bhi[q] = fmax(bhi[q], mi[k].hi[q]);
            }
            gmn = min(gmn, mi[k].gmin);
            gmx = max(gmx, mi[k].gmax);
        }
        const double cells = (double)kI * 32.0;
        for (int sl = 0; sl < nslab; ++sl) {
            const SlabMeta &mj = meta[h0 / 32 + sl];
            if (!both) {
                c += c_diag * cells;
                continue;
            }
            const bool fast = (mj.gmax < gmn || mj.gmin > gmx) &&
                              (boxes_far(blo, bhi, mj) || islabs_far<TBI>(mi, kvalid, mj));
            c += (fast ? 1.0 : c_checked) * cells;
        }
    }
    cost[t] = c;
}

__constant__ int d_capsules_off;   // SF_SYM_CAPSULE=0 (A/B measurements)

// Read SF_SYM_CAPSULE once per process, before the first slab-meta launch
// (never inside a stream capture: the first call runs uncaptured).
static void ensure_capsule_flag() {
    static const bool done = [] {
        const char *e = getenv("SF_SYM_CAPSULE");
        const int off = (e && atoi(e) == 0) ? 1 : 0;
        cudaMemcpyToSymbol(d_capsules_off, &off, sizeof(int));
        return true;
    }();
    (void)done;
}

// Capsule of one 32-point slab from every lane's point (valid lanes first):
// p0 = the slab's first point, p1 = its last valid point, rad = the largest
// point-to-segment distance (padded up for rounding).
__device__ __forceinline__ void slab_capsule(const double *pt, bool valid, int nvalid, SlabMeta &m) {
    const int lane = threadIdx.x & 31;
    double p0[3], p1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        p0[c] = __shfl_sync(0xffffffffu, pt[c], 0);
        p1[c] = __shfl_sync(0xffffffffu, pt[c], nvalid - 1);
    }
    double d = 0.0;
    if (valid) d = sqrt(seg_seg_dist2(pt, pt, p0, p1));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (lane == 0) {
        for (int c = 0; c < 3; ++c) { m.p0[c] = p0[c]; m.p1[c] = p1[c]; }
        m.rad = d_capsules_off ? -1.0 : d * (1.0 + 1e-12) + 1e-14;
    }
}

// The slab's common doublet coefficient (lane 0 is always a real point), NaN
// when its real points differ.
__device__ __forceinline__ double slab_common_c(double c, bool valid) {
    const double c0 = __shfl_sync(0xffffffffu, c, 0);
    const bool same = __all_sync(0xffffffffu, !valid || c == c0);
    return same ? c0 : __longlong_as_double(0x7ff8000000000000ll);
}

__global__ void slab_meta_kernel(const SymSrc *__restrict__ src, int64_t N,
                                 SlabMeta *__restrict__ meta) {
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s * 32 >= N) return;
    const int64_t j = s * 32 + lane;
    double v[6], pt[3] = {0.0, 0.0, 0.0}, cj = 0.0;
    int gmn = 0x7fffffff, gmx = (int)0x80000000;
    if (j < N) {
        const SymSrc &q = src[j];
        v[0] = v[3] = pt[0] = q.v[0];
        v[1] = v[4] = pt[1] = q.v[1];
        v[2] = v[5] = pt[2] = q.v[2];
        cj = q.v[6];
        if (q.g >= 0) { gmn = q.g; gmx = q.g; }
    } else {
        v[0] = v[1] = v[2] = 1e300;
        v[3] = v[4] = v[5] = -1e300;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            v[c] = fmin(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
            v[3 + c] = fmax(v[3 + c], __shfl_xor_sync(0xffffffffu, v[3 + c], o));
        }
        gmn = min(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
        gmx = max(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
    }
    SlabMeta m;
    slab_capsule(pt, j < N, (int)min((int64_t)32, N - s * 32), m);
    const double cu = slab_common_c(cj, j < N);
    if (lane == 0) {
        for (int c = 0; c < 3; ++c) { m.lo[c] = v[c]; m.hi[c] = v[3 + c]; }
        m.gmin = gmn;
        m.gmax = gmx;
        m.cuni = cu;
        meta[s] = m;
    }
}


// ------------------------------------------------ FP32-compute variant ----
// Same task structure; pair arithmetic in FP32, FP32 sums over one 32-point
// slab, FP64 accumulation across slabs (owner sums in registers, transposed
// sums in shared memory).
//
// Positions are slab-relative: every 32-point slab has an FP64 origin o_s
// (its bounding-box centre) and a record stores float(y - o_s).  For a j
// slab the i points are re-expressed once, in FP64, relative to that slab's
// origin: xr_i = float((x_i - o_i) + (o_i - o_j)), so each pair costs a single
// FP32 subtraction per component, r = xr_i - yl_j.  Both operands are small
// whenever r is small (|xr_i| <= r + slab extent), so the rounding error of
// r stays at FP32 precision relative to r itself -- the property the earlier
// hi+lo split bought with three subtractions per component.
// Record floats: ylx yly ylz fx fy fz c c3 (32 bytes), int g at the record's end.
struct PDataF {
    float x, y, z, fx, fy, fz, c, c3;
    int g;
};

__device__ __forceinline__ float rsqrt_ftz(float x) {
    // every fast-path r^2 is >= 1e-20 > FLT_MIN; checked pairs select 0 for r^2 < 1e-24
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ PDataF load_point_f(const SymSrc *src, int64_t k, bool valid) {
    PDataF p;
    if (valid) {
        const float4 *q = reinterpret_cast<const float4 *>(src + k);
        const float4 a0 = q[0], a1 = q[1];
        p.x = a0.x; p.y = a0.y; p.z = a0.z; p.fx = a0.w;
        p.fy = a1.x; p.fz = a1.y; p.c = a1.z; p.c3 = a1.w;
        p.g = src[k].g;
    } else {  // strengthless and far away (padding i lanes sit at +1e18 instead,
              // so no two padding points coincide; r^2 stays finite in FP32)
        p.x = p.y = p.z = -1e18f;
        p.fx = p.fy = p.fz = p.c = p.c3 = 0.f;
        p.g = -3;
    }
    return p;
}

__device__ __forceinline__ void slab_origin(const SlabMeta &m, double *o) {
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] = 0.5 * (m.lo[c] + m.hi[c]);
}

// CHECK: group exclusion, and the r^2 < 1e-24 skip decided on the FP64
// positions (slab-relative FP32 coordinates of coincident points in
// different slabs round differently, so FP32 r would not be exactly 0).
template <bool CHECK, bool BOTH>
__device__ __forceinline__ void sym_pair_f(const PDataF &pi, const PDataF &pj, float *ui,
                                           float *uj, int &nb, const double *xi = nullptr,
                                           const double *xj = nullptr) {
    const float rx = pi.x - pj.x, ry = pi.y - pj.y, rz = pi.z - pj.z;
    const float r2 = fmaf(rx, rx, fmaf(ry, ry, rz * rz));
    float ir = rsqrt_ftz(r2);
    if (CHECK) {
        const bool excl = (pi.g == pj.g) && pi.g >= 0;
        bool small = false;
        if (xi && xj && !excl) {
            const double dx = xi[0] - xj[0], dy = xi[1] - xj[1], dz = xi[2] - xj[2];
            small = below_min_sep(fma(dx, dx, fma(dy, dy, dz * dz)));
        }
        nb += (small && !excl) ? (BOTH ? 2 : 1) : 0;
        ir = (excl || small) ? 0.f : ir;
    }
    const float ir2 = ir * ir;
    const float ir3 = ir * ir2;
    const float ir5 = ir3 * ir2;
    {
        const float a = fmaf(pj.c, ir3, ir);
        const float b = fmaf(rz, pj.fz, fmaf(ry, pj.fy, rx * pj.fx)) * fmaf(-pj.c3, ir5, ir3);
        ui[0] = fmaf(a, pj.fx, fmaf(b, rx, ui[0]));
        ui[1] = fmaf(a, pj.fy, fmaf(b, ry, ui[1]));
        ui[2] = fmaf(a, pj.fz, fmaf(b, rz, ui[2]));
    }
    if (BOTH) {
        const float a = fmaf(pi.c, ir3, ir);
        const float b = fmaf(rz, pi.fz, fmaf(ry, pi.fy, rx * pi.fx)) * fmaf(-pi.c3, ir5, ir3);
        uj[0] = fmaf(a, pi.fx, fmaf(b, rx, uj[0]));
        uj[1] = fmaf(a, pi.fy, fmaf(b, ry, uj[1]));
        uj[2] = fmaf(a, pi.fz, fmaf(b, rz, uj[2]));
    }
}

// FP32 form of sym_step_grouped (fast path, both directions), phase by phase
// so the shared j operands come from the operand reuse cache.
template <int TBI>
__device__ __forceinline__ void sym_step_grouped_f(const PDataF (&pi)[TBI], const PDataF &pj,
                                                   float (&ui)[TBI][3], float *uj) {
    float rx[TBI], ry[TBI], rz[TBI], ir[TBI], ir3[TBI], ir5[TBI];
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        rx[q] = pi[q].x - pj.x;
        ry[q] = pi[q].y - pj.y;
        rz[q] = pi[q].z - pj.z;
    }
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        ir[q] = rsqrt_ftz(fmaf(rx[q], rx[q], fmaf(ry[q], ry[q], rz[q] * rz[q])));
        const float ir2 = ir[q] * ir[q];
        ir3[q] = ir[q] * ir2;
        ir5[q] = ir3[q] * ir2;
    }
    float a[TBI], b[TBI];
#pragma unroll
    for (int q = 0; q < TBI; ++q) a[q] = fmaf(pj.c, ir3[q], ir[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = rx[q] * pj.fx;
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = fmaf(ry[q], pj.fy, b[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] = fmaf(rz[q], pj.fz, b[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) b[q] *= fmaf(-pj.c3, ir5[q], ir3[q]);
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][0] = fmaf(a[q], pj.fx, fmaf(b[q], rx[q], ui[q][0]));
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][1] = fmaf(a[q], pj.fy, fmaf(b[q], ry[q], ui[q][1]));
#pragma unroll
    for (int q = 0; q < TBI; ++q) ui[q][2] = fmaf(a[q], pj.fz, fmaf(b[q], rz[q], ui[q][2]));
#pragma unroll
    for (int q = 0; q < TBI; ++q) {
        const float ai = fmaf(pi[q].c, ir3[q], ir[q]);
        const float bi = fmaf(rz[q], pi[q].fz, fmaf(ry[q], pi[q].fy, rx[q] * pi[q].fx)) *
                         fmaf(-pi[q].c3, ir5[q], ir3[q]);
        uj[0] = fmaf(ai, pi[q].fx, fmaf(bi, rx[q], uj[0]));
        uj[1] = fmaf(ai, pi[q].fy, fmaf(bi, ry[q], uj[1]));
        uj[2] = fmaf(ai, pi[q].fz, fmaf(bi, rz[q], uj[2]));
    }
}

template <int MINB, int TBI>
__global__ void __launch_bounds__(kSymThreads, MINB) sym_task_kernel_f32(SymArgs a) {
    constexpr int kI = 32 * TBI;
    extern __shared__ double jacc_s[];
    __shared__ double ui_s[4][kI][3];
    __shared__ float4 js_a[4][32], js_b[4][32];
    __shared__ int js_g[4][32];
    if ((int64_t)blockIdx.x >= a.ntasks) return;
    const int64_t t = a.task0 + blockIdx.x;
    int g, h;
    task_units(t, a.G, g, h);
    const bool both = g != h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t)g * a.M, h0 = (int64_t)h * a.M;
    const int ng = (int)min((int64_t)a.M, a.N - g0), nh = (int)min((int64_t)a.M, a.N - h0);
    const int nslab = (nh + 31) / 32;
    if (both)
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x) jacc_s[e] = 0.0;
    __syncthreads();   // zero-fill (any warp) before the owning warp's first +=
    int nb = 0;
    for (int ib = 0; ib < ng; ib += kI) {
        PDataF pi[TBI];
        float xl[TBI][3];    // own-slab-relative positions
        double oi[TBI][3];   // own slab origins
        bool vi[TBI];
        double ud[TBI][3];
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            vi[k] = ib + 32 * k + lane < ng;
            pi[k] = load_point_f(a.src, g0 + ib + 32 * k + lane, vi[k]);
            xl[k][0] = pi[k].x; xl[k][1] = pi[k].y; xl[k][2] = pi[k].z;
            const int64_t sk = (g0 + ib) / 32 + (vi[k] ? k : 0);
            slab_origin(a.slab[sk], oi[k]);
            ud[k][0] = ud[k][1] = ud[k][2] = 0.0;
        }
        const SlabMeta *mi = a.slab + (g0 + ib) / 32;
        const int kvalid = min(TBI, (ng - ib + 31) / 32);
        double blo[3], bhi[3];
        int gmn = mi[0].gmin, gmx = mi[0].gmax;
        for (int c = 0; c < 3; ++c) { blo[c] = mi[0].lo[c]; bhi[c] = mi[0].hi[c]; }
        for (int k = 1; k < kvalid; ++k) {
            for (int c = 0; c < 3; ++c) {
                blo[c] = fmin(blo[c], mi[k].lo[c]);
                bhi[c] = fmax(bhi[c], mi[k].hi[c]);
            }
            gmn = min(gmn, mi[k].gmin);
            gmx = max(gmx, mi[k].gmax);
        }
        for (int sl = warp; sl < nslab; sl += 4) {
            const int jl = sl * 32 + lane;
            {
                const PDataF q = load_point_f(a.src, h0 + jl, jl < nh);
                js_a[warp][lane] = make_float4(q.x, q.y, q.z, q.fx);
                js_b[warp][lane] = make_float4(q.fy, q.fz, q.c, q.c3);
                js_g[warp][lane] = q.g;
            }
            const SlabMeta &mj = a.slab[h0 / 32 + sl];
            {   // i points relative to this j slab's origin (FP64, once per slab);
                // padding i lanes sit 1e18 away and carry no strength
                double oj[3];
                slab_origin(mj, oj);
#pragma unroll
                for (int k = 0; k < TBI; ++k) {
                    pi[k].x = vi[k] ? (float)(((double)xl[k][0] + (oi[k][0] - oj[0]))) : 1e18f;
                    pi[k].y = vi[k] ? (float)(((double)xl[k][1] + (oi[k][1] - oj[1]))) : 1e18f;
                    pi[k].z = vi[k] ? (float)(((double)xl[k][2] + (oi[k][2] - oj[2]))) : 1e18f;
                }
            }
            __syncwarp();
            float uf[TBI][3];
#pragma unroll
            for (int k = 0; k < TBI; ++k) uf[k][0] = uf[k][1] = uf[k][2] = 0.f;
            float uj[3] = {0.f, 0.f, 0.f};
            const bool fast = !a.nofast && (mj.gmax < gmn || mj.gmin > gmx) &&
                              (boxes_far(blo, bhi, mj) || islabs_far<TBI>(mi, kvalid, mj));
            const int nxt = (lane + 1) & 31;
            if (fast && both) {
#pragma unroll 4
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PDataF pj;
                    const float4 A0 = js_a[warp][k], B0 = js_b[warp][k];
                    pj.x = A0.x; pj.y = A0.y; pj.z = A0.z; pj.fx = A0.w;
                    pj.fy = B0.x; pj.fz = B0.y; pj.c = B0.z; pj.c3 = B0.w;
                    pj.g = 0;
                    sym_step_grouped_f<TBI>(pi, pj, uf, uj);
                    uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                    uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                    uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                }
            } else {
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PDataF pj;
                    const float4 A0 = js_a[warp][k], B0 = js_b[warp][k];
                    pj.x = A0.x; pj.y = A0.y; pj.z = A0.z; pj.fx = A0.w;
                    pj.fy = B0.x; pj.fz = B0.y; pj.c = B0.z; pj.c3 = B0.w;
                    pj.g = js_g[warp][k];
                    int nbi = 0;
                    if (fast) {
#pragma unroll
                        for (int q = 0; q < TBI; ++q) sym_pair_f<false, false>(pi[q], pj, uf[q], uj, nbi);
                    } else {
                        const double *xj = pj.g != -3 ? a.x + 3 * (h0 + sl * 32 + k) : nullptr;
#pragma unroll
                        for (int q = 0; q < TBI; ++q) {
                            const double *xi = vi[q] ? a.x + 3 * (g0 + ib + 32 * q + lane) : nullptr;
                            if (both) sym_pair_f<true, true>(pi[q], pj, uf[q], uj, nbi, xi, xj);
                            else sym_pair_f<true, false>(pi[q], pj, uf[q], uj, nbi, xi, xj);
                        }
                    }
                    if (pj.g != -3) nb += nbi;
                    if (both) {
                        uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                        uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                        uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < TBI; ++k) {
                ud[k][0] += (double)uf[k][0];
                ud[k][1] += (double)uf[k][1];
                ud[k][2] += (double)uf[k][2];
            }
            if (both && jl < nh) {
                double *dst = jacc_s + 3 * jl;
                dst[0] += (double)uj[0];
                dst[1] += (double)uj[1];
                dst[2] += (double)uj[2];
            }
        }
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            ui_s[warp][32 * k + lane][0] = ud[k][0];
            ui_s[warp][32 * k + lane][1] = ud[k][1];
            ui_s[warp][32 * k + lane][2] = ud[k][2];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * kI; e += blockDim.x) {
            const int il = e / 3, c = e - 3 * il;
            if (ib + il < ng) {
                const double sv = ((ui_s[0][il][c] + ui_s[1][il][c]) + ui_s[2][il][c]) + ui_s[3][il][c];
                part_store(a, owner_slot(a, g, h, ib + il) + c, sv);
            }
        }
        __syncthreads();
    }
    if (both) {
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x)
            part_store(a, trans_slot(a, g, h0) + e, jacc_s[e]);
    }
    if (a.bad) {
        nb = warp_sum_int(nb);
        if (lane == 0 && nb) atomicAdd(a.bad, (unsigned long long)nb);
    }
}

// ---------------------------------------------------------------------------
// Packed FP32c variant: the check-free both-direction slab pairs run on
// packed FP32 (FFMA2 / FADD2 / FMUL2, two lanes of arithmetic per issue slot).
// The FP32c kernel above is issue-bound (19.3 SASS instructions per pair
// interaction, FP32 pipe ~59 % busy); here the packing is over TWO j points
// against one i point, so nothing is broadcast inside the loop: a j slab of
// 32 points is staged in shared memory as 16 pairs {j, j + 16} (positions
// negated, so r = x_i + (-y_j) is the same FP32 subtraction as above), each
// half-warp rotates the 16 pairs among its 16 lanes, and a pair's transposed
// accumulator is one float2 per component -- 6 shuffles per step for 2 j
// points, the same shuffle count per interaction as the scalar kernel.  The
// i operands are duplicated into both halves of a register pair once per
// slab.  After the 16 steps the two half-warps' transposed partials are
// added with one xor-16 shuffle, and each i point's two packed halves once.
// Per step and i point: 33 packed FP32 instructions + 2 MUFU for 4 pair
// interactions.  Checked and diagonal slab pairs use the scalar path.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 dup2(float a) { return make_float2(a, a); }

template <int TBI, bool GROUPED, bool JUNI>
__device__ __forceinline__ void sym_slab_packed(const float4 (*__restrict__ jp)[16], int lane,
                                                float cjf, float nc3jf,
                                                const float2 (&ix)[TBI], const float2 (&iy)[TBI],
                                                const float2 (&iz)[TBI], const float2 (&ifx)[TBI],
                                                const float2 (&ify)[TBI], const float2 (&ifz)[TBI],
                                                const float2 (&ic)[TBI], const float2 (&inc3)[TBI],
                                                float (&uf)[TBI][3], float (&ujo)[3]) {
    float2 ua[TBI][3], uj[3];
#pragma unroll
    for (int q = 0; q < TBI; ++q) ua[q][0] = ua[q][1] = ua[q][2] = f2(0.f, 0.f);
    uj[0] = uj[1] = uj[2] = f2(0.f, 0.f);
    const int half = lane & 16, l = lane & 15;
    const int nxt = half | ((l + 1) & 15);
#pragma unroll 2
    for (int s = 0; s < 16; ++s) {
        const int p = (l + s) & 15;
        const float4 A = jp[0][p], B = jp[1][p], C = jp[2][p];
        const float2 nxj = f2(A.x, A.y), nyj = f2(A.z, A.w), nzj = f2(B.x, B.y);
        const float2 fxj = f2(B.z, B.w), fyj = f2(C.x, C.y), fzj = f2(C.z, C.w);
        float2 cj, nc3j;
        if (JUNI) {   // one c for the whole j slab: a 32-bit broadcast operand
            cj = dup2(cjf); nc3j = dup2(nc3jf);
        } else {
            const float4 D = jp[3][p];
            cj = f2(D.x, D.y); nc3j = f2(D.z, D.w);
        }
        if (GROUPED) {   // phase by phase over the i points: independent work between
                         // each MUFU / FFMA2 and its first use
            float2 rx[TBI], ry[TBI], rz[TBI], ir[TBI], ir3[TBI], ir5[TBI];
#pragma unroll
            for (int q = 0; q < TBI; ++q) {
                rx[q] = __fadd2_rn(ix[q], nxj);
                ry[q] = __fadd2_rn(iy[q], nyj);
                rz[q] = __fadd2_rn(iz[q], nzj);
            }
#pragma unroll
            for (int q = 0; q < TBI; ++q) {
                const float2 r2 =
                    __ffma2_rn(rx[q], rx[q], __ffma2_rn(ry[q], ry[q], __fmul2_rn(rz[q], rz[q])));
                ir[q] = f2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
            }
#pragma unroll
            for (int q = 0; q < TBI; ++q) {
                const float2 ir2 = __fmul2_rn(ir[q], ir[q]);
                ir3[q] = __fmul2_rn(ir[q], ir2);
                ir5[q] = __fmul2_rn(ir3[q], ir2);
            }
#pragma unroll
            for (int q = 0; q < TBI; ++q) {   // the two j sources onto i
                const float2 a = __ffma2_rn(cj, ir3[q], ir[q]);
                const float2 rf =
                    __ffma2_rn(rz[q], fzj, __ffma2_rn(ry[q], fyj, __fmul2_rn(rx[q], fxj)));
                const float2 b = __fmul2_rn(rf, __ffma2_rn(nc3j, ir5[q], ir3[q]));
                ua[q][0] = __ffma2_rn(a, fxj, __ffma2_rn(b, rx[q], ua[q][0]));
                ua[q][1] = __ffma2_rn(a, fyj, __ffma2_rn(b, ry[q], ua[q][1]));
                ua[q][2] = __ffma2_rn(a, fzj, __ffma2_rn(b, rz[q], ua[q][2]));
            }
#pragma unroll
            for (int q = 0; q < TBI; ++q) {   // i onto the two j targets
                const float2 a = __ffma2_rn(ic[q], ir3[q], ir[q]);
                const float2 rf = __ffma2_rn(rz[q], ifz[q],
                                             __ffma2_rn(ry[q], ify[q], __fmul2_rn(rx[q], ifx[q])));
                const float2 b = __fmul2_rn(rf, __ffma2_rn(inc3[q], ir5[q], ir3[q]));
                uj[0] = __ffma2_rn(a, ifx[q], __ffma2_rn(b, rx[q], uj[0]));
                uj[1] = __ffma2_rn(a, ify[q], __ffma2_rn(b, ry[q], uj[1]));
                uj[2] = __ffma2_rn(a, ifz[q], __ffma2_rn(b, rz[q], uj[2]));
            }
        } else {
#pragma unroll
            for (int q = 0; q < TBI; ++q) {
                const float2 rx = __fadd2_rn(ix[q], nxj);
                const float2 ry = __fadd2_rn(iy[q], nyj);
                const float2 rz = __fadd2_rn(iz[q], nzj);
                const float2 r2 = __ffma2_rn(rx, rx, __ffma2_rn(ry, ry, __fmul2_rn(rz, rz)));
                const float2 ir = f2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
                const float2 ir2 = __fmul2_rn(ir, ir);
                const float2 ir3 = __fmul2_rn(ir, ir2);
                const float2 ir5 = __fmul2_rn(ir3, ir2);
                {   // the two j sources onto i
                    const float2 a = __ffma2_rn(cj, ir3, ir);
                    const float2 rf = __ffma2_rn(rz, fzj, __ffma2_rn(ry, fyj, __fmul2_rn(rx, fxj)));
                    const float2 b = __fmul2_rn(rf, __ffma2_rn(nc3j, ir5, ir3));
                    ua[q][0] = __ffma2_rn(a, fxj, __ffma2_rn(b, rx, ua[q][0]));
                    ua[q][1] = __ffma2_rn(a, fyj, __ffma2_rn(b, ry, ua[q][1]));
                    ua[q][2] = __ffma2_rn(a, fzj, __ffma2_rn(b, rz, ua[q][2]));
                }
                {   // i onto the two j targets
                    const float2 a = __ffma2_rn(ic[q], ir3, ir);
                    const float2 rf =
                        __ffma2_rn(rz, ifz[q], __ffma2_rn(ry, ify[q], __fmul2_rn(rx, ifx[q])));
                    const float2 b = __fmul2_rn(rf, __ffma2_rn(inc3[q], ir5, ir3));
                    uj[0] = __ffma2_rn(a, ifx[q], __ffma2_rn(b, rx, uj[0]));
                    uj[1] = __ffma2_rn(a, ify[q], __ffma2_rn(b, ry, uj[1]));
                    uj[2] = __ffma2_rn(a, ifz[q], __ffma2_rn(b, rz, uj[2]));
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            uj[c].x = __shfl_sync(0xffffffffu, uj[c].x, nxt);
            uj[c].y = __shfl_sync(0xffffffffu, uj[c].y, nxt);
        }
    }
    // lane l of each half now holds pair l = {j = l, j = l + 16}, summed over
    // its half's i points; the sum of both halves is the same in both (a + b)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float ox = __shfl_xor_sync(0xffffffffu, uj[c].x, 16);
        const float oy = __shfl_xor_sync(0xffffffffu, uj[c].y, 16);
        ujo[c] = half ? uj[c].y + oy : uj[c].x + ox;
    }
#pragma unroll
    for (int q = 0; q < TBI; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) uf[q][c] = ua[q][c].x + ua[q][c].y;
}

template <int MINB, int TBI, bool GROUPED = false, bool UDS = false>
__global__ void __launch_bounds__(kSymThreads, MINB) sym_task_kernel_f32p(SymArgs a) {
    constexpr int kI = 32 * TBI;
    extern __shared__ double jacc_s[];
    __shared__ double ui_s[4][kI][3];
    __shared__ float4 js_a[4][32], js_b[4][32];
    __shared__ int js_g[4][32];
    __shared__ float4 jp_s[4][4][16];   // [warp][record quarter][pair]: a half-warp's LDS.128 of
                                        // one quarter reads 16 consecutive float4 (no bank
                                        // conflicts; [pair][quarter] cost 4 wavefronts per load)
    if ((int64_t)blockIdx.x >= a.ntasks) return;
    const int64_t t = a.task0 + blockIdx.x;
    int g, h;
    task_units(t, a.G, g, h);
    const bool both = g != h;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g0 = (int64_t)g * a.M, h0 = (int64_t)h * a.M;
    const int ng = (int)min((int64_t)a.M, a.N - g0), nh = (int)min((int64_t)a.M, a.N - h0);
    const int nslab = (nh + 31) / 32;
    if (both)
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x) jacc_s[e] = 0.0;
    __syncthreads();   // zero-fill (any warp) before the owning warp's first +=
    int nb = 0;
    for (int ib = 0; ib < ng; ib += kI) {
        // i strengths, duplicated into both halves of a register pair
        float2 ifx[TBI], ify[TBI], ifz[TBI], ic[TBI], inc3[TBI];
        bool vi[TBI];
        double ud[TBI][3];
#pragma unroll
        for (int k = 0; k < TBI; ++k) {
            vi[k] = ib + 32 * k + lane < ng;
            const PDataF p = load_point_f(a.src, g0 + ib + 32 * k + lane, vi[k]);
            ifx[k] = dup2(p.fx); ify[k] = dup2(p.fy); ifz[k] = dup2(p.fz);
            ic[k] = dup2(p.c); inc3[k] = dup2(-p.c3);
            if constexpr (UDS) {   // FP64 owner sums in this warp's shared rows (registers
                                   // for the packed loop)
                ui_s[warp][32 * k + lane][0] = ui_s[warp][32 * k + lane][1] =
                    ui_s[warp][32 * k + lane][2] = 0.0;
            } else {
                ud[k][0] = ud[k][1] = ud[k][2] = 0.0;
            }
        }
        const SlabMeta *mi = a.slab + (g0 + ib) / 32;
        const int kvalid = min(TBI, (ng - ib + 31) / 32);
        double blo[3], bhi[3];
        int gmn = mi[0].gmin, gmx = mi[0].gmax;
        for (int c = 0; c < 3; ++c) { blo[c] = mi[0].lo[c]; bhi[c] = mi[0].hi[c]; }
        for (int k = 1; k < kvalid; ++k) {
            for (int c = 0; c < 3; ++c) {
                blo[c] = fmin(blo[c], mi[k].lo[c]);
                bhi[c] = fmax(bhi[c], mi[k].hi[c]);
            }
            gmn = min(gmn, mi[k].gmin);
            gmx = max(gmx, mi[k].gmax);
        }
        for (int sl = warp; sl < nslab; sl += 4) {
            const int jl = sl * 32 + lane;
            const PDataF qj = load_point_f(a.src, h0 + jl, jl < nh);
            const SlabMeta &mj = a.slab[h0 / 32 + sl];
            const bool fast = !a.nofast && both && (mj.gmax < gmn || mj.gmin > gmx) &&
                              (boxes_far(blo, bhi, mj) || islabs_far<TBI>(mi, kvalid, mj));
            // i points relative to this j slab's origin (FP64 positions, once
            // per slab); padding i lanes sit 1e18 away and carry no strength
            double oj[3];
            slab_origin(mj, oj);
            float px[TBI], py[TBI], pz[TBI];
#pragma unroll
            for (int k = 0; k < TBI; ++k) {
                const double *xi = a.x + 3 * (g0 + ib + 32 * k + (vi[k] ? lane : 0));
                px[k] = vi[k] ? (float)(xi[0] - oj[0]) : 1e18f;
                py[k] = vi[k] ? (float)(xi[1] - oj[1]) : 1e18f;
                pz[k] = vi[k] ? (float)(xi[2] - oj[2]) : 1e18f;
            }
            float uf[TBI][3];
            float uj[3] = {0.f, 0.f, 0.f};
            if (fast) {
                {   // stage the slab as 16 pairs {p, p + 16}
                    float *d = reinterpret_cast<float *>(&jp_s[warp][0][lane & 15]) + (lane >> 4);
                    d[0] = -qj.x; d[2] = -qj.y; d[64] = -qj.z; d[66] = qj.fx;
                    d[128] = qj.fy; d[130] = qj.fz; d[192] = qj.c; d[194] = -qj.c3;
                }
                __syncwarp();
                float2 ix[TBI], iy[TBI], iz[TBI];
#pragma unroll
                for (int k = 0; k < TBI; ++k) { ix[k] = dup2(px[k]); iy[k] = dup2(py[k]); iz[k] = dup2(pz[k]); }
                // records hold float(c), float(3c): the same roundings here
                const float cjf = __double2float_rn(mj.cuni);
                const float nc3jf = -__double2float_rn(3.0 * mj.cuni);
                if (mj.cuni == mj.cuni)   // not NaN: the slab's points share c
                    sym_slab_packed<TBI, GROUPED, true>(jp_s[warp], lane, cjf, nc3jf, ix, iy, iz, ifx,
                                                        ify, ifz, ic, inc3, uf, uj);
                else
                    sym_slab_packed<TBI, GROUPED, false>(jp_s[warp], lane, cjf, nc3jf, ix, iy, iz,
                                                         ifx, ify, ifz, ic, inc3, uf, uj);
            } else {
                js_a[warp][lane] = make_float4(qj.x, qj.y, qj.z, qj.fx);
                js_b[warp][lane] = make_float4(qj.fy, qj.fz, qj.c, qj.c3);
                js_g[warp][lane] = qj.g;
                __syncwarp();
                PDataF pi[TBI];
#pragma unroll
                for (int k = 0; k < TBI; ++k) {
                    pi[k].x = px[k]; pi[k].y = py[k]; pi[k].z = pz[k];
                    pi[k].fx = ifx[k].x; pi[k].fy = ify[k].x; pi[k].fz = ifz[k].x;
                    pi[k].c = ic[k].x; pi[k].c3 = -inc3[k].x;
                    pi[k].g = vi[k] ? a.src[g0 + ib + 32 * k + lane].g : -3;
                    uf[k][0] = uf[k][1] = uf[k][2] = 0.f;
                }
                const int nxt = (lane + 1) & 31;
                for (int s = 0; s < 32; ++s) {
                    const int k = (lane + s) & 31;
                    PDataF pj;
                    const float4 A0 = js_a[warp][k], B0 = js_b[warp][k];
                    pj.x = A0.x; pj.y = A0.y; pj.z = A0.z; pj.fx = A0.w;
                    pj.fy = B0.x; pj.fz = B0.y; pj.c = B0.z; pj.c3 = B0.w;
                    pj.g = js_g[warp][k];
                    int nbi = 0;
                    const double *xj = pj.g != -3 ? a.x + 3 * (h0 + sl * 32 + k) : nullptr;
#pragma unroll
                    for (int q = 0; q < TBI; ++q) {
                        const double *xi = vi[q] ? a.x + 3 * (g0 + ib + 32 * q + lane) : nullptr;
                        if (both) sym_pair_f<true, true>(pi[q], pj, uf[q], uj, nbi, xi, xj);
                        else sym_pair_f<true, false>(pi[q], pj, uf[q], uj, nbi, xi, xj);
                    }
                    if (pj.g != -3) nb += nbi;
                    if (both) {
                        uj[0] = __shfl_sync(0xffffffffu, uj[0], nxt);
                        uj[1] = __shfl_sync(0xffffffffu, uj[1], nxt);
                        uj[2] = __shfl_sync(0xffffffffu, uj[2], nxt);
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < TBI; ++k) {
                if constexpr (UDS) {
                    double *d = ui_s[warp][32 * k + lane];
                    d[0] += (double)uf[k][0];
                    d[1] += (double)uf[k][1];
                    d[2] += (double)uf[k][2];
                } else {
                    ud[k][0] += (double)uf[k][0];
                    ud[k][1] += (double)uf[k][1];
                    ud[k][2] += (double)uf[k][2];
                }
            }
            if (both && jl < nh) {
                double *dst = jacc_s + 3 * jl;
                dst[0] += (double)uj[0];
                dst[1] += (double)uj[1];
                dst[2] += (double)uj[2];
            }
        }
        if constexpr (!UDS) {
#pragma unroll
            for (int k = 0; k < TBI; ++k) {
                ui_s[warp][32 * k + lane][0] = ud[k][0];
                ui_s[warp][32 * k + lane][1] = ud[k][1];
                ui_s[warp][32 * k + lane][2] = ud[k][2];
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * kI; e += blockDim.x) {
            const int il = e / 3, c = e - 3 * il;
            if (ib + il < ng) {
                const double sv = ((ui_s[0][il][c] + ui_s[1][il][c]) + ui_s[2][il][c]) + ui_s[3][il][c];
                part_store(a, owner_slot(a, g, h, ib + il) + c, sv);
            }
        }
        __syncthreads();
    }
    if (both) {
        __syncthreads();
        for (int e = threadIdx.x; e < 3 * nh; e += blockDim.x)
            part_store(a, trans_slot(a, g, h0) + e, jacc_s[e]);
    }
    if (a.bad) {
        nb = warp_sum_int(nb);
        if (lane == 0 && nb) atomicAdd(a.bad, (unsigned long long)nb);
    }
}

// Slab bounds straight from the FP64 positions (the FP32 records are packed
// relative to these boxes' centres afterwards).
__global__ void slab_meta_x_kernel(const double *__restrict__ x, const int64_t *__restrict__ grp,
                                   const double *__restrict__ dcoef, int64_t N,
                                   SlabMeta *__restrict__ meta) {
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s * 32 >= N) return;
    const int64_t j = s * 32 + lane;
    double v[6];
    int gmn = 0x7fffffff, gmx = (int)0x80000000;
    double pt[3] = {0.0, 0.0, 0.0};
    if (j < N) {
        for (int c = 0; c < 3; ++c) v[c] = v[3 + c] = pt[c] = x[3 * j + c];
        const int gj = grp ? pack_source_group(grp[j]) : -1;
        if (gj >= 0) { gmn = gj; gmx = gj; }
    } else {
        v[0] = v[1] = v[2] = 1e300;
        v[3] = v[4] = v[5] = -1e300;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            v[c] = fmin(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
            v[3 + c] = fmax(v[3 + c], __shfl_xor_sync(0xffffffffu, v[3 + c], o));
        }
        gmn = min(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
        gmx = max(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
    }
    SlabMeta m;
    slab_capsule(pt, j < N, (int)min((int64_t)32, N - s * 32), m);
    const double cu = slab_common_c((dcoef && j < N) ? dcoef[j] : 0.0, j < N);
    if (lane == 0) {
        for (int c = 0; c < 3; ++c) { m.lo[c] = v[c]; m.hi[c] = v[3 + c]; }
        m.gmin = gmn;
        m.gmax = gmx;
        m.cuni = cu;
        meta[s] = m;
    }
}

// FP32 record packing: float positions relative to the slab origin, weighted
// strengths, c, 3c.
__global__ void sym_pack_f32_kernel(const double *__restrict__ x, const int64_t *__restrict__ grp,
                                    const double *__restrict__ f, const double *__restrict__ w,
                                    const double *__restrict__ dcoef, int64_t N,
                                    const SlabMeta *__restrict__ meta, SymSrc *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x) {
        SymSrc s;
        float *pf = reinterpret_cast<float *>(&s);
        double o[3];
        slab_origin(meta[j / 32], o);
        const double wj = w ? w[j] : 1.0;
        for (int c = 0; c < 3; ++c) {
            pf[c] = __double2float_rn(x[3 * j + c] - o[c]);
            pf[3 + c] = __double2float_rn(wj * f[3 * j + c]);
        }
        const double c = dcoef ? dcoef[j] : 0.0;
        pf[6] = __double2float_rn(c);
        pf[7] = __double2float_rn(3.0 * c);
        for (int k = 8; k < 18; ++k) pf[k] = 0.f;
        s.g = grp ? pack_source_group(grp[j]) : -1;
        s.pad = 0;
        out[j] = s;
    }
}

__device__ __forceinline__ int64_t task_index(int64_t g, int64_t h, int64_t G) {
    return g * G - g * (g - 1) / 2 + (h - g);
}

// acc[i] += this wave's partials of point i, in slot order: the transposed
// slots k in [ga, min(gl, u - 1)] (tasks {k, u}), then, when u is one of the
// wave's rows, the owner slots h >= u (tasks {u, h}); only tasks inside the
// wave's range [tb, te) (a partial first or last row, a rank's share) count.
// The task index grows along both slot runs, so the counted slots are one
// contiguous run each; their loads are issued 8 at a time (independent) and
// added in slot order, so the sum is the same as one load per add (the
// serial form ran latency-bound: 51 us at C2 for 67 MB).
__device__ __forceinline__ double strided_sum(double s, const double *__restrict__ q,
                                              int64_t stride, int64_t n) {
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcs(q + (i + j) * stride);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; i < n; ++i) s += __ldcs(q + i * stride);
    return s;
}

__global__ void sym_wave_reduce_kernel(const double *__restrict__ A, const double *__restrict__ B,
                                       int G, int64_t N, int M, int64_t ga, int64_t gl,
                                       int64_t tb, int64_t te, int64_t Acols, int64_t Bstride,
                                       double *__restrict__ acc) {
    const int64_t e = 3 * ga * M + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 3 * N) return;
    const int64_t p = e / 3, c = e - 3 * p;
    const int64_t u = p / M;
    double s = acc[e];
    int64_t k0 = ga, k1 = min(gl, u - 1);
    while (k0 <= k1 && task_index(k0, u, G) < tb) ++k0;
    while (k1 >= k0 && task_index(k1, u, G) >= te) --k1;
    if (k1 >= k0)
        s = strided_sum(s, B + ((k0 - ga) * Bstride + (p - ga * M)) * 3 + c, Bstride * 3, k1 - k0 + 1);
    if (u >= ga && u <= gl) {
        const int64_t loc = p - u * M;
        int64_t h0 = u, h1 = G - 1;
        while (h0 <= h1 && task_index(u, h0, G) < tb) ++h0;
        while (h1 >= h0 && task_index(u, h1, G) >= te) --h1;
        if (h1 >= h0)
            s = strided_sum(s, A + (((u - ga) * Acols + (h0 - ga)) * M + loc) * 3 + c,
                            (int64_t)M * 3, h1 - h0 + 1);
    }
    acc[e] = s;
}

// out[i] (+)= pref * acc[i]
__global__ void sym_scale_kernel(const double *__restrict__ acc, int64_t n, double pref,
                                 double *__restrict__ out, int accumulate) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    out[e] = accumulate ? out[e] + pref * acc[e] : pref * acc[e];
}

// Packing identical to the pair engine's (x y z, w f, c, 3c, group).
__global__ void sym_pack_kernel(const double *__restrict__ x, const int64_t *__restrict__ grp,
                                const double *__restrict__ f, const double *__restrict__ w,
                                const double *__restrict__ dcoef, int64_t N,
                                SymSrc *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x) {
        SymSrc s;
        const double wj = w ? w[j] : 1.0;
        s.v[0] = x[3 * j]; s.v[1] = x[3 * j + 1]; s.v[2] = x[3 * j + 2];
        s.v[3] = wj * f[3 * j]; s.v[4] = wj * f[3 * j + 1]; s.v[5] = wj * f[3 * j + 2];
        const double c = dcoef ? dcoef[j] : 0.0;
        s.v[6] = c; s.v[7] = 3.0 * c; s.v[8] = 0.0;
        s.g = grp ? pack_source_group(grp[j]) : -1;
        s.pad = 0;
        out[j] = s;
    }
}

int sym_unit_size(int64_t N, int64_t group_size, int mode) {
    // units: a multiple of the 32-point slab (and of the fiber size when that
    // keeps them near the target, so units align to fibers), at most 3072
    // points in FP64 (1408 for FP32c, whose 4 CTAs/SM need the smaller
    // M x 3 shared accumulator: 1.478e12 pair/s at C5 against 1.420e12 with
    // 1536 points, where shared memory allows only 3), and small enough that the G(G+1)/2 unit-pair
    // tasks fill the GPU many times over (G >= 128 -> >= 8256 tasks) for
    // mid-size systems; the sweeps (tools/gpu_unit_sweep.sh) peak at
    // N/128..N/85 for N = 32k-64k, and at C5 M = 3072 matches 2048 (750 vs
    // 748 G/s) with a third fewer partial slots (8.6 instead of 12.9 GB)
    const char *e = getenv("SF_SYM_UNIT");
    int64_t target = e ? atoi(e) : (mode == SF_MODE_FP32C ? 1408 : 3072);
    if (!e) {
        const int64_t fill = N / 128;
        if (fill < target) target = fill;
        if (target < 256) target = 256;
        // r02 sweep (tools/gpu_r02_unit.sh): at N = 32,768 (C2) 384-point
        // units beat 256 by 2.2 % (1.653 vs 1.690 ms) and still give 7 waves
        // of tasks; at N = 65,536 (C4 fibers) N/128 = 512 stays best
        if (N >= 24576 && target < 384) target = 384;
    }
    // multiple of the 128-point i-sub-block (4 per lane x 32 lanes) so no
    // sub-block runs part-empty, and of the fiber size when possible
    target = (target / 128) * 128;
    if (target < 128) target = 128;
    if (group_size > 0) {
        int64_t a = group_size, b = 128;
        while (b) { const int64_t t = a % b; a = b; b = t; }
        const int64_t l = group_size / a * 128;  // lcm(group_size, 128)
        if (l <= target) return (int)((target / l) * l);
    }
    return (int)target;
}

// mode SF_MODE_FP64 picks the symmetric evaluation for large enough blocks;
// SF_MODE_FP64_DIRECT forces the per-target order of the reference.
bool use_symmetric(int mode, int64_t N) {
    if (mode != SF_MODE_FP64 && mode != SF_MODE_FP32C) return false;
    const char *e = getenv("SF_SYMMETRIC");
    if (e && atoi(e) == 0) return false;
    return N >= 8192;
}

int pairs_sbt_symmetric(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                        const double *f, const double *w, const double *dcoef, double pref,
                        double *out, int64_t *bad, int accumulate, cudaStream_t st,
                        Workspace &ws, int mode, const std::function<int()> *after_pack) {
    return pairs_sbt_symmetric_shard(x, grp, N, group_size, f, w, dcoef, pref, 0, 1, out, bad,
                                     accumulate, st, ws, mode, after_pack);
}

// The unit-pair tasks of rank `rank` of `world`: out receives this rank's
// contribution to EVERY point; summing `out` over ranks (reduce-scatter)
// gives the full sum.
// Contiguous task range of `rank`, balanced by pair count: task {g,h}
// evaluates n_g n_h pair geometries in both directions (cost 2 n_g n_h), a
// diagonal task n_g^2 ordered pairs; unit sizes n_g = min(M, N - g M) (the
// last unit may be ragged).  Tasks run row by row, each row
// g = {g,g}, {g,g+1}, ..., {g,G-1} starting with its diagonal.
int64_t sym_task_range(int64_t G, int64_t N, int64_t M, int rank, int world, int64_t *count) {
    const int64_t ntasks = G * (G + 1) / 2;
    auto nu = [&](int64_t g) { return std::min(M, N - g * M); };
    // suffix sums of unit sizes and prefix costs of whole rows
    std::vector<int64_t> suffix(G + 1, 0), rowpre(G + 1, 0);
    for (int64_t g = G - 1; g >= 0; --g) suffix[g] = suffix[g + 1] + nu(g);
    for (int64_t g = 0; g < G; ++g)
        rowpre[g + 1] = rowpre[g] + nu(g) * nu(g) + 2 * nu(g) * suffix[g + 1];
    auto start = [&](int64_t row) { return row * G - row * (row - 1) / 2; };
    auto boundary = [&](int r) {   // first task whose prefix cost reaches r/world of the total
        if (r <= 0) return (int64_t)0;
        if (r >= world) return ntasks;
        const int64_t total = rowpre[G];
        const int64_t want = total / world * r + (total % world) * r / world;
        // row holding the boundary: rowpre[g] < want <= rowpre[g + 1]
        int64_t g = std::upper_bound(rowpre.begin(), rowpre.end(), want - 1) - rowpre.begin() - 1;
        if (g < 0) g = 0;
        if (g >= G) return ntasks;
        int64_t c = rowpre[g], t = start(g);
        if (c >= want) return t;
        c += nu(g) * nu(g);                 // the diagonal task
        ++t;
        for (int64_t h = g + 1; h < G && c < want; ++h, ++t) c += 2 * nu(g) * nu(h);
        return t;
    };
    const int64_t b = boundary(rank), e = boundary(rank + 1);
    *count = e - b;
    return b;
}

struct SymWave {
    int64_t tb, te, ga, gl;
};

// partial-buffer budget per wave and number of wave buffers/streams:
// SF_SYM_WAVE_MB / SF_SYM_STREAMS at first use, or sf_sym_set_waves()
static int64_t g_wave_bytes = -1;
static int g_wave_streams = -1;

size_t sym_wave_bytes() {
    if (g_wave_bytes < 0) {
        const char *e = getenv("SF_SYM_WAVE_MB");
        g_wave_bytes = (int64_t)((e ? atof(e) : 192.0) * (double)(1 << 20));
    }
    return (size_t)g_wave_bytes;
}

int sym_wave_streams() {
    if (g_wave_streams < 0) {
        const char *e = getenv("SF_SYM_STREAMS");
        g_wave_streams = e ? atoi(e) : 2;
    }
    return std::max(1, std::min(g_wave_streams, SidePool::kStreams));
}

void sym_set_waves(int64_t bytes, int streams) {
    g_wave_bytes = bytes > 0 ? bytes : -1;
    g_wave_streams = streams > 0 ? streams : -1;
}

// Waves over the task range [t0, t1): whole task rows from the first row of
// the wave, as many as fit `budget` bytes of partials (at least one row).
// Row g needs (G - ga) M + (N - ga M) points x 3 doubles, so a wave holds a
// roughly constant number of tasks (budget / (2 M x 24 bytes)).
static std::vector<SymWave> sym_waves(int64_t G, int64_t N, int64_t M, int64_t t0, int64_t t1,
                                      size_t budget, size_t *max_bytes) {
    std::vector<SymWave> out;
    *max_bytes = 0;
    auto start = [&](int64_t row) { return row * G - row * (row - 1) / 2; };
    int64_t t = t0, row = 0;
    while (t < t1) {
        while (row + 1 < G && start(row + 1) <= t) ++row;
        const int64_t ga = row;
        const size_t per_row = (size_t)((G - ga) * M + (N - ga * M)) * 3 * sizeof(double);
        int64_t rows = (int64_t)(budget / per_row);
        if (rows < 1) rows = 1;
        const int64_t gl = std::min(G - 1, ga + rows - 1);
        const int64_t te = std::min(t1, start(gl + 1));
        out.push_back({t, te, ga, gl});
        *max_bytes = std::max(*max_bytes, (size_t)(gl - ga + 1) * per_row);
        t = te;
    }
    return out;
}

int pairs_sbt_symmetric_shard(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                              const double *f, const double *w, const double *dcoef, double pref,
                              int rank, int world, double *out, int64_t *bad, int accumulate,
                              cudaStream_t st, Workspace &ws, int mode,
                              const std::function<int()> *after_pack) {
    int64_t ntasks = 0, t0 = 0;
    if (N > 0) {
        const int M = sym_unit_size(N, group_size, mode);
        const int G = (int)((N + M - 1) / M);
        t0 = sym_task_range(G, N, M, rank, world, &ntasks);
    }
    return pairs_sbt_symmetric_tasks(x, grp, N, group_size, f, w, dcoef, pref, t0, ntasks, out, bad,
                                     accumulate, st, ws, mode, after_pack);
}

int64_t sym_task_total(int64_t N, int64_t group_size, int mode) {
    if (N <= 0) return 0;
    const int64_t M = sym_unit_size(N, group_size, mode);
    const int64_t G = (N + M - 1) / M;
    return G * (G + 1) / 2;
}

int sym_task_costs(const double *x, const int64_t *grp, int64_t N, int64_t group_size, int mode,
                   double c_checked, double c_diag, double *cost, cudaStream_t st, Workspace &ws) {
    if (N == 0) return SF_OK;
    ensure_capsule_flag();
    const int M = sym_unit_size(N, group_size, mode);
    const int G = (int)((N + M - 1) / M);
    const int64_t ntasks = (int64_t)G * (G + 1) / 2;
    const int64_t nslab = (N + 31) / 32;
    SlabMeta *meta = (SlabMeta *)ws.get(4, sizeof(SlabMeta) * (size_t)(nslab + 1), st);
    if (!meta) return SF_ENOMEM;
    slab_meta_x_kernel<<<(unsigned)((nslab + 7) / 8), 256, 0, st>>>(x, grp, nullptr, N, meta);
    sym_task_cost_kernel<<<(unsigned)((ntasks + 127) / 128), 128, 0, st>>>(meta, N, M, G, ntasks,
                                                                         c_checked, c_diag, cost);
    return check_launch("sym_task_cost_kernel");
}

// The unit-pair tasks [t0, t0 + ntasks) (any contiguous range: a rank's
// share): out receives their contribution to every point.  `after_pack`
// (optional) runs once the packing kernels are queued and before the task
// kernel: the operator forks its overlapping side-stream work there, so the
// short packing kernels are not held up behind it.
int pairs_sbt_symmetric_tasks(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                              const double *f, const double *w, const double *dcoef, double pref,
                              int64_t t0, int64_t ntasks, double *out, int64_t *bad,
                              int accumulate, cudaStream_t st, Workspace &ws, int mode,
                              const std::function<int()> *after_pack) {
    const bool f32 = mode == SF_MODE_FP32C;
    if (bad && cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess)
        return check_launch("memset");
    if (N == 0) return (after_pack && *after_pack) ? (*after_pack)() : SF_OK;
    ensure_capsule_flag();
    const int M = sym_unit_size(N, group_size, mode);
    const int G = (int)((N + M - 1) / M);
    if (t0 < 0 || ntasks < 0 || t0 + ntasks > (int64_t)G * (G + 1) / 2)
        return set_error(SF_EINVAL, "task range outside the %lld unit-pair tasks",
                         (long long)((int64_t)G * (G + 1) / 2));
    const size_t wave_bytes = sym_wave_bytes();
    const int nbuf_env = sym_wave_streams();
    size_t buf_bytes = 0;
    const std::vector<SymWave> waves = sym_waves(G, N, M, t0, t0 + ntasks, wave_bytes, &buf_bytes);
    SidePool *pool = (waves.size() > 1 && nbuf_env > 1) ? side_pool_for(st) : nullptr;
    const int nbuf = pool ? (int)std::min<size_t>(nbuf_env, waves.size()) : 1;
    buf_bytes = (buf_bytes + 255) / 256 * 256;

    SymSrc *packed = (SymSrc *)ws.get(3, sizeof(SymSrc) * (size_t)N, st);
    SlabMeta *meta = (SlabMeta *)ws.get(4, sizeof(SlabMeta) * (size_t)((N + 31) / 32 + 1), st);
    double *acc = (double *)ws.get(5, sizeof(double) * 3 * (size_t)N, st);
    char *bufs = (char *)ws.get(12, buf_bytes * nbuf, st);
    if (!packed || !meta || !acc || (!bufs && !waves.empty())) return SF_ENOMEM;
    if (cudaMemsetAsync(acc, 0, sizeof(double) * 3 * (size_t)N, st) != cudaSuccess)
        return check_launch("memset");
    int64_t pg = (N + 255) / 256;
    const int64_t nslab = (N + 31) / 32;
    if (f32) {
        slab_meta_x_kernel<<<(unsigned)((nslab + 7) / 8), 256, 0, st>>>(x, grp, dcoef, N, meta);
        sym_pack_f32_kernel<<<(unsigned)(pg > 4096 ? 4096 : pg), 256, 0, st>>>(x, grp, f, w, dcoef,
                                                                             N, meta, packed);
    } else {
        sym_pack_kernel<<<(unsigned)(pg > 4096 ? 4096 : pg), 256, 0, st>>>(x, grp, f, w, dcoef, N,
                                                                         packed);
        slab_meta_kernel<<<(unsigned)((nslab + 7) / 8), 256, 0, st>>>(packed, N, meta);
    }
    int rc = check_launch("sym_pack");
    if (rc) return rc;
    if (after_pack && *after_pack && (rc = (*after_pack)())) return rc;
    SymArgs a;
    a.src = packed;
    a.slab = meta;
    a.N = N;
    a.M = M;
    a.G = G;
    a.bad = (unsigned long long *)bad;
    a.x = x;
    static const int nofast = [] {
        const char *e = getenv("SF_SYM_NOFAST");
        return e ? atoi(e) : 0;
    }();
    a.nofast = nofast;
    static const double l2_keep_mb = [] {   // SF_SYM_L2_MB: largest wave kept in L2
        const char *e = getenv("SF_SYM_L2_MB");
        return e ? atof(e) : 80.0;
    }();
    const double l2_keep = l2_keep_mb * (double)(1 << 20);
    const size_t smem = sizeof(double) * 3 * M;
    static const int variant = [] {  // tuning knob: MINB*10 + i-per-lane
        const char *e = getenv("SF_SYM_VARIANT");
        return e ? atoi(e) : 224;
    }();
    static const int fvariant = [] {
        const char *e = getenv("SF_SYM_F32_VARIANT");
        return e ? atoi(e) : 344;   // packed, grouped, owner sums in shared memory, 4 CTAs/SM
    }();
    auto launch = [&](auto kern, cudaStream_t s) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return check_launch("cudaFuncSetAttribute");
        if (a.ntasks > 0) kern<<<(unsigned)a.ntasks, kSymThreads, smem, s>>>(a);
        return check_launch("sym_task_kernel");
    };
    auto run = [&](cudaStream_t s) -> int {
        if (f32) {
            switch (fvariant) {
                case 24: return launch(sym_task_kernel_f32<2, 4>, s);
                case 33: return launch(sym_task_kernel_f32<3, 3>, s);
                case 26: return launch(sym_task_kernel_f32<2, 6>, s);
                case 44: return launch(sym_task_kernel_f32<4, 4>, s);
                case 134: return launch(sym_task_kernel_f32p<3, 4>, s);
                case 124: return launch(sym_task_kernel_f32p<2, 4>, s);
                case 133: return launch(sym_task_kernel_f32p<3, 3>, s);
                case 142: return launch(sym_task_kernel_f32p<4, 2>, s);
                case 234: return launch(sym_task_kernel_f32p<3, 4, true>, s);
                case 224: return launch(sym_task_kernel_f32p<2, 4, true>, s);
                case 233: return launch(sym_task_kernel_f32p<3, 3, true>, s);
                case 334: return launch(sym_task_kernel_f32p<3, 4, true, true>, s);
                case 344: return launch(sym_task_kernel_f32p<4, 4, true, true>, s);
                case 343: return launch(sym_task_kernel_f32p<4, 3, true, true>, s);
                case 444: return launch(sym_task_kernel_f32p<4, 4, false, true>, s);
                default: return launch(sym_task_kernel_f32<3, 4>, s);
            }
        }
        switch (variant) {
            // launch-shape sweep (tools/gpu_sym_sweep.sh, tools/gpu_sym_aster_sweep.sh):
            // MINB*10 + i-per-lane (+100 prefetch, +200 prefetch + grouped pairs)
            case 24: return launch(sym_task_kernel<2, 4>, s);
            case 124: return launch(sym_task_kernel<2, 4, true>, s);
            case 233: return launch(sym_task_kernel<3, 3, true, true>, s);
            case 223: return launch(sym_task_kernel<2, 3, true, true>, s);
            case 232: return launch(sym_task_kernel<3, 2, true, true>, s);
            default: return launch(sym_task_kernel<2, 4, true, true>, s);   // 749 G/s at C5
        }
    };
    // fork the side streams off the caller's stream (packed sources, slab
    // metas and the zeroed sums are ready)
    if (pool) {
        if (cudaEventRecord(pool->fork, st) != cudaSuccess) return check_launch("event record");
        for (int b = 1; b < nbuf; ++b)
            if (cudaStreamWaitEvent(pool->s[b - 1], pool->fork, 0) != cudaSuccess)
                return check_launch("stream wait");
    }
    int prev = -1;   // buffer (stream) of the previous wave's ordered reduce
    for (size_t wv = 0; wv < waves.size(); ++wv) {
        const SymWave &W = waves[wv];
        const int b = (int)(wv % nbuf);
        cudaStream_t s = b == 0 ? st : pool->s[b - 1];
        double *A = (double *)(bufs + (size_t)b * buf_bytes);
        const int64_t rows = W.gl - W.ga + 1;
        a.task0 = W.tb;
        a.ntasks = W.te - W.tb;
        a.ga = W.ga;
        a.Acols = G - W.ga;
        a.Bstride = N - W.ga * M;
        a.partA = A;
        a.partB = A + (size_t)rows * a.Acols * M * 3;
        // bytes of partials the wave writes (two M-point slices per task)
        a.cs = (double)a.ntasks * 2.0 * M * 3 * sizeof(double) > l2_keep ? 1 : 0;
        if ((rc = run(s))) return rc;
        // the running sums are added to in wave order
        if (prev >= 0 && prev != b && cudaStreamWaitEvent(s, pool->done[prev], 0) != cudaSuccess)
            return check_launch("stream wait");
        const int64_t nel = 3 * (N - W.ga * M);
        sym_wave_reduce_kernel<<<(unsigned)((nel + 255) / 256), 256, 0, s>>>(
            a.partA, a.partB, G, N, M, W.ga, W.gl, W.tb, W.te, a.Acols, a.Bstride, acc);
        if ((rc = check_launch("sym_wave_reduce_kernel"))) return rc;
        if (pool && cudaEventRecord(pool->done[b], s) != cudaSuccess)
            return check_launch("event record");
        prev = b;
    }
    // join: the last reduce waited on every earlier one
    if (pool && prev > 0 && cudaStreamWaitEvent(st, pool->done[prev], 0) != cudaSuccess)
        return check_launch("stream wait");
    sym_scale_kernel<<<(unsigned)((3 * N + 255) / 256), 256, 0, st>>>(acc, 3 * N, pref, out,
                                                                     accumulate);
    return check_launch("sym_scale_kernel");
}

// kernels launched by one pairs_sbt_symmetric_tasks call over [t0, t0 + ntasks)
int64_t sym_launch_count_range(int64_t N, int64_t group_size, int mode, int64_t t0,
                               int64_t ntasks) {
    if (N == 0) return 0;
    const int M = sym_unit_size(N, group_size, mode);
    const int64_t G = (N + M - 1) / M;
    size_t mx = 0;
    const auto w = sym_waves(G, N, M, t0, t0 + ntasks, sym_wave_bytes(), &mx);
    return 3 + 2 * (int64_t)w.size();   // pack + meta + per wave (tasks + reduce) + scale
}

// kernels launched by one pairs_sbt_symmetric_shard call (gpu_launches accounting)
int64_t sym_launch_count(int64_t N, int64_t group_size, int mode, int rank, int world) {
    if (N == 0) return 0;
    const int M = sym_unit_size(N, group_size, mode);
    const int64_t G = (N + M - 1) / M;
    int64_t ntasks = 0;
    const int64_t t0 = sym_task_range(G, N, M, rank, world, &ntasks);
    return sym_launch_count_range(N, group_size, mode, t0, ntasks);
}

}  // namespace sf
