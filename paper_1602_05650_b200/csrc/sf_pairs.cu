// sf_pairs.cu — all-pairs target x source kernels of the HI operator, sm_100a.
//
// One engine, four physics policies:
//   SbtP<DBL>      Stokeslet (+ (eps L)^2/2 source doublet), FP64      kernels.py:72-145
//   SbtF32cP       the same in FP32 arithmetic with FP64 accumulation (north_star variant)
//   StressletP     off-surface double layer                             kernels.py:177-213
//   DlSubP         on-surface singularity-subtracted double layer       kernels.py:216-249
//   RowsumP        per-node 3x3 stresslet row sums                      kernels.py:252-281
//
// Engine (pair_kernel): a CTA owns NT*TB consecutive targets (TB per thread,
// strided by NT so the one-time target loads coalesce) and streams a
// contiguous source range through shared memory in TS-source tiles.  Each
// tile is one 1-D bulk async copy (cp.async.bulk -> TMA engine, SASS UBLKCP)
// completing on an mbarrier, double buffered so tile t+1 lands while tile t
// is consumed.  Every thread reads the same source at the same time (smem
// broadcast, no bank conflicts), so the inner loop is pure FP64-pipe work:
// per pair r (3 DADD), r^2 (3), rsqrt (MUFU.RSQ64H seed + 5-op cubic
// correction), then the physics.  Group exclusion and the r^2 < 1e-24 skip
// are branch-free: they zero the rsqrt seed, which makes the pair's
// contribution exactly +0 (a skipped term, as in the reference), and the
// skipped-and-not-excluded pairs are counted in integer registers.
//
// Determinism: each target's sum runs over its source range in index order;
// with a source split (blockIdx.y) the per-chunk partials are summed in chunk
// order by reduce_partials.  The split factor depends only on (nt, ns), never
// on the device, so results are bitwise reproducible.
#include <cstdlib>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

struct __align__(16) Src80 {
    double v[9];
    int g;
    int pad;
};
static_assert(sizeof(Src80) == 80, "packed source must be 80 bytes");

struct PairArgs {
    const double *trg;      // (nt,3)
    const int64_t *tgrp;    // (nt) or nullptr (no exclusion)
    const double *tq;       // (nt,3) target densities (DlSub) or nullptr
    int64_t nt;
    const Src80 *src;       // packed sources
    int64_t ns;
    int64_t chunk;          // sources per blockIdx.y
    double pref;
    double *out;            // final output (nsplit == 1)
    double *partial;        // (nsplit, nt, NOUT) unscaled partials (nsplit > 1)
    unsigned long long *bad;
    int nsplit;
    int accumulate;         // out += result instead of out = result
};

// ---------------------------------------------------------------- physics ----
struct TargetBase {
    double x, y, z;
    int g;
};

__device__ __forceinline__ void load_target_base(const PairArgs &a, int64_t i, TargetBase &t,
                                                 bool by_index) {
    t.x = a.trg[3 * i + 0];
    t.y = a.trg[3 * i + 1];
    t.z = a.trg[3 * i + 2];
    if (by_index)
        t.g = (int)i;
    else
        t.g = a.tgrp ? pack_target_group(a.tgrp[i]) : kNoGroup;
}

// Every policy also exposes target_pos (FP64 coordinates, for the CTA box),
// target_group (the id compared with source groups; < 0 = none) and
// kFloatPositions (packed positions are float hi/lo pairs).
__device__ __forceinline__ void target_xyz(const PairArgs &a, int64_t i, double *x) {
    x[0] = a.trg[3 * i];
    x[1] = a.trg[3 * i + 1];
    x[2] = a.trg[3 * i + 2];
}

// Stokeslet + optional doublet.  Source slots: x y z fx fy fz c 3c.
template <bool DBL>
struct SbtP {
    static constexpr int NACC = 3;
    static constexpr int NOUT = 3;
    static constexpr bool kBad = true;
    static constexpr bool kFloatPositions = false;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    typedef TargetBase Target;
    struct SrcR {
        double x, y, z, fx, fy, fz, c, c3;
        int g;
    };
    typedef double TAcc[3];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        load_target_base(a, i, t, false);
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) {
        const double2 *p = reinterpret_cast<const double2 *>(&s);
        double2 a0 = p[0], a1 = p[1], a2 = p[2];
        r.x = a0.x; r.y = a0.y; r.z = a1.x; r.fx = a1.y; r.fy = a2.x; r.fz = a2.y;
        if (DBL) {
            double2 a3 = p[3];
            r.c = a3.x; r.c3 = a3.y;
        }
        r.g = s.g;
    }
    __device__ static void zero(TAcc &t) { t[0] = t[1] = t[2] = 0.0; }
    __device__ static void flush(TAcc &, double *) {}
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &, double *u,
                                                int &nb) {
        const double rx = t.x - s.x, ry = t.y - s.y, rz = t.z - s.z;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq_seed(r2);
        if (CHECK) {
            const bool excl = (s.g == t.g);
            const bool small = below_min_sep(r2);
            nb += (small && !excl) ? 1 : 0;
            y0 = (excl || small) ? 0.0 : y0;
        }
        const double ir = rsq_refine(r2, y0);
        const double ir2 = ir * ir;
        const double ir3 = ir * ir2;
        const double rf = fma(rx, s.fx, fma(ry, s.fy, rz * s.fz));
        double a, bb;
        if (DBL) {
            const double ir5 = ir3 * ir2;
            a = fma(s.c, ir3, ir);       // 1/r + c/r^3
            bb = fma(-s.c3, ir5, ir3);   // 1/r^3 - 3c/r^5
        } else {
            a = ir;
            bb = ir3;
        }
        const double b = rf * bb;
        u[0] = fma(a, s.fx, u[0]);
        u[1] = fma(a, s.fy, u[1]);
        u[2] = fma(a, s.fz, u[2]);
        u[0] = fma(b, rx, u[0]);
        u[1] = fma(b, ry, u[1]);
        u[2] = fma(b, rz, u[2]);
    }

    // Check-free lockstep form for TB targets: each stage is issued for all
    // targets back to back so the source operand (c, 3c, f) they share sits in
    // the same slot of consecutive DFMAs (register reuse cache: one fresh
    // operand read instead of two).
    template <int TB>
    __device__ __forceinline__ static void pair_fast(const Target *t, const SrcR &s,
                                                     double (*u)[3]) {
        double rx[TB], ry[TB], rz[TB], r2[TB], y[TB], a[TB], bb[TB], rf[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            rx[k] = t[k].x - s.x;
            ry[k] = t[k].y - s.y;
            rz[k] = t[k].z - s.z;
        }
#pragma unroll
        for (int k = 0; k < TB; ++k) r2[k] = fma(rx[k], rx[k], fma(ry[k], ry[k], rz[k] * rz[k]));
#pragma unroll
        for (int k = 0; k < TB; ++k) y[k] = rsq_refine(r2[k], rsq_seed(r2[k]));
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            const double ir2 = y[k] * y[k];
            const double ir3 = y[k] * ir2;
            if (DBL) {
                const double ir5 = ir3 * ir2;
                a[k] = ir3;
                bb[k] = ir5;
            } else {
                a[k] = y[k];
                bb[k] = ir3;
            }
        }
        if (DBL) {
#pragma unroll
            for (int k = 0; k < TB; ++k) bb[k] = fma(-s.c3, bb[k], a[k]);  // 1/r^3 - 3c/r^5
#pragma unroll
            for (int k = 0; k < TB; ++k) a[k] = fma(s.c, a[k], y[k]);      // 1/r + c/r^3
        }
#pragma unroll
        for (int k = 0; k < TB; ++k) rf[k] = rx[k] * s.fx;
#pragma unroll
        for (int k = 0; k < TB; ++k) rf[k] = fma(ry[k], s.fy, rf[k]);
#pragma unroll
        for (int k = 0; k < TB; ++k) rf[k] = fma(rz[k], s.fz, rf[k]);
#pragma unroll
        for (int k = 0; k < TB; ++k) rf[k] = rf[k] * bb[k];
#pragma unroll
        for (int k = 0; k < TB; ++k) u[k][0] = fma(a[k], s.fx, u[k][0]);
#pragma unroll
        for (int k = 0; k < TB; ++k) u[k][1] = fma(a[k], s.fy, u[k][1]);
#pragma unroll
        for (int k = 0; k < TB; ++k) u[k][2] = fma(a[k], s.fz, u[k][2]);
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            u[k][0] = fma(rf[k], rx[k], u[k][0]);
            u[k][1] = fma(rf[k], ry[k], u[k][1]);
            u[k][2] = fma(rf[k], rz[k], u[k][2]);
        }
    }
};

// Dispatch of the check-free inner step: lockstep form where a policy has
// one, else the per-target pair.
template <class P, int TB>
struct FastStep {
    __device__ __forceinline__ static void run(const typename P::Target *tg,
                                               const typename P::SrcR &sr, typename P::TAcc *ta,
                                               double (*u)[P::NACC], int *nb) {
#pragma unroll
        for (int k = 0; k < TB; ++k) P::template pair<false>(tg[k], sr, ta[k], u[k], nb[k]);
    }
};
template <bool DBL, int TB>
struct FastStep<SbtP<DBL>, TB> {
    __device__ __forceinline__ static void run(const TargetBase *tg,
                                               const typename SbtP<DBL>::SrcR &sr, double (*)[3],
                                               double (*u)[3], int *) {
        SbtP<DBL>::template pair_fast<TB>(tg, sr, u);
    }
};

// Doublet alone (kernels.py:114-145).  Source slots: x y z fx fy fz.
struct DoubletP {
    static constexpr int NACC = 3;
    static constexpr int NOUT = 3;
    static constexpr bool kBad = true;
    static constexpr bool kFloatPositions = false;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    typedef TargetBase Target;
    typedef typename SbtP<false>::SrcR SrcR;
    typedef double TAcc[1];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        load_target_base(a, i, t, false);
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) { SbtP<false>::load_src(s, r); }
    __device__ static void zero(TAcc &) {}
    __device__ static void flush(TAcc &, double *) {}
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &, double *u,
                                                int &nb) {
        const double rx = t.x - s.x, ry = t.y - s.y, rz = t.z - s.z;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq_seed(r2);
        if (CHECK) {
            const bool excl = (s.g == t.g);
            const bool small = below_min_sep(r2);
            nb += (small && !excl) ? 1 : 0;
            y0 = (excl || small) ? 0.0 : y0;
        }
        const double ir = rsq_refine(r2, y0);
        const double ir2 = ir * ir;
        const double ir3 = ir * ir2;
        const double ir5 = ir3 * ir2;
        const double rf = fma(rx, s.fx, fma(ry, s.fy, rz * s.fz));
        const double b = -3.0 * rf * ir5;
        u[0] = fma(ir3, s.fx, fma(b, rx, u[0]));
        u[1] = fma(ir3, s.fy, fma(b, ry, u[1]));
        u[2] = fma(ir3, s.fz, fma(b, rz, u[2]));
    }
};

// FP32-compute / FP64-accumulate Stokeslet + doublet.  Positions are split
// into float hi + lo parts so r = (t_hi - s_hi) + (t_lo - s_lo) keeps FP32
// relative accuracy in r even when |r| << |x|.  Per-tile FP32 partial sums
// are flushed into FP64 accumulators once per tile.
// Source float slots: xh yh zh xl yl zl fx fy fz c c3 (11 floats) + g.
struct SbtF32cP {
    static constexpr int NACC = 3;
    static constexpr int NOUT = 3;
    static constexpr bool kBad = true;
    static constexpr bool kFloatPositions = true;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    struct Target {
        float xh, yh, zh, xl, yl, zl;
        int g;
    };
    struct SrcR {
        float xh, yh, zh, xl, yl, zl, fx, fy, fz, c, c3;
        int g;
    };
    typedef float TAcc[3];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        const double x = a.trg[3 * i + 0], y = a.trg[3 * i + 1], z = a.trg[3 * i + 2];
        t.xh = __double2float_rn(x); t.xl = __double2float_rn(x - (double)t.xh);
        t.yh = __double2float_rn(y); t.yl = __double2float_rn(y - (double)t.yh);
        t.zh = __double2float_rn(z); t.zl = __double2float_rn(z - (double)t.zh);
        t.g = a.tgrp ? pack_target_group(a.tgrp[i]) : kNoGroup;
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) {
        const float4 *p = reinterpret_cast<const float4 *>(&s);
        float4 a0 = p[0], a1 = p[1], a2 = p[2];
        r.xh = a0.x; r.yh = a0.y; r.zh = a0.z; r.xl = a0.w;
        r.yl = a1.x; r.zl = a1.y; r.fx = a1.z; r.fy = a1.w;
        r.fz = a2.x; r.c = a2.y; r.c3 = a2.z;
        r.g = s.g;
    }
    __device__ static void zero(TAcc &t) { t[0] = t[1] = t[2] = 0.f; }
    __device__ static void flush(TAcc &t, double *u) {
        u[0] += (double)t[0]; u[1] += (double)t[1]; u[2] += (double)t[2];
        t[0] = t[1] = t[2] = 0.f;
    }
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &ta, double *,
                                                int &nb) {
        const float rx = (t.xh - s.xh) + (t.xl - s.xl);
        const float ry = (t.yh - s.yh) + (t.yl - s.yl);
        const float rz = (t.zh - s.zh) + (t.zl - s.zl);
        const float r2 = fmaf(rx, rx, fmaf(ry, ry, rz * rz));
        float ir = rsqrtf(r2);
        if (CHECK) {
            const bool excl = (s.g == t.g);
            // same skip rule, evaluated on the FP32 r^2 (1e-24 is a normal float)
            const bool small = r2 < 1e-24f;
            nb += (small && !excl) ? 1 : 0;
            ir = (excl || small) ? 0.f : ir;
        }
        const float ir2 = ir * ir;
        const float ir3 = ir * ir2;
        const float ir5 = ir3 * ir2;
        const float rf = fmaf(rx, s.fx, fmaf(ry, s.fy, rz * s.fz));
        const float a = fmaf(s.c, ir3, ir);
        const float b = rf * fmaf(-s.c3, ir5, ir3);
        ta[0] = fmaf(a, s.fx, fmaf(b, rx, ta[0]));
        ta[1] = fmaf(a, s.fy, fmaf(b, ry, ta[1]));
        ta[2] = fmaf(a, s.fz, fmaf(b, rz, ta[2]));
    }
};

// Off-surface stresslet.  Source slots: x y z nx ny nz qx qy qz.
struct StressletP {
    static constexpr int NACC = 3;
    static constexpr int NOUT = 3;
    static constexpr bool kBad = true;
    static constexpr bool kFloatPositions = false;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    typedef TargetBase Target;
    struct SrcR {
        double x, y, z, nx, ny, nz, qx, qy, qz;
        int g;
    };
    typedef double TAcc[1];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        load_target_base(a, i, t, false);
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) {
        r.x = s.v[0]; r.y = s.v[1]; r.z = s.v[2];
        r.nx = s.v[3]; r.ny = s.v[4]; r.nz = s.v[5];
        r.qx = s.v[6]; r.qy = s.v[7]; r.qz = s.v[8];
        r.g = s.g;
    }
    __device__ static void zero(TAcc &) {}
    __device__ static void flush(TAcc &, double *) {}
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &, double *u,
                                                int &nb) {
        const double rx = t.x - s.x, ry = t.y - s.y, rz = t.z - s.z;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq_seed(r2);
        if (CHECK) {
            const bool excl = (s.g == t.g);
            const bool small = below_min_sep(r2);
            nb += (small && !excl) ? 1 : 0;
            y0 = (excl || small) ? 0.0 : y0;
        }
        const double ir = rsq_refine(r2, y0);
        const double ir2 = ir * ir;
        const double ir5 = ir * ir2 * ir2;
        const double qr = fma(s.qx, rx, fma(s.qy, ry, s.qz * rz));
        const double nr = fma(s.nx, rx, fma(s.ny, ry, s.nz * rz));
        const double c = qr * nr * ir5;
        u[0] = fma(c, rx, u[0]);
        u[1] = fma(c, ry, u[1]);
        u[2] = fma(c, rz, u[2]);
    }
};

// On-surface subtracted double layer.  Source slots: x y z (w n)xyz qx qy qz,
// g = node index (j == i excluded).  Target carries q_i.
struct DlSubP {
    static constexpr int NACC = 3;
    static constexpr int NOUT = 3;
    static constexpr bool kBad = false;  // the reference has no skip rule here
    static constexpr bool kFloatPositions = false;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    struct Target {
        double x, y, z, qx, qy, qz;
        int g;
    };
    struct SrcR {
        double x, y, z, nx, ny, nz, qx, qy, qz;
        int g;
    };
    typedef double TAcc[1];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        t.x = a.trg[3 * i + 0]; t.y = a.trg[3 * i + 1]; t.z = a.trg[3 * i + 2];
        t.qx = a.tq[3 * i + 0]; t.qy = a.tq[3 * i + 1]; t.qz = a.tq[3 * i + 2];
        t.g = (int)i;
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) {
        r.x = s.v[0]; r.y = s.v[1]; r.z = s.v[2];
        r.nx = s.v[3]; r.ny = s.v[4]; r.nz = s.v[5];
        r.qx = s.v[6]; r.qy = s.v[7]; r.qz = s.v[8];
        r.g = s.g;
    }
    __device__ static void zero(TAcc &) {}
    __device__ static void flush(TAcc &, double *) {}
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &, double *u,
                                                int &) {
        const double rx = t.x - s.x, ry = t.y - s.y, rz = t.z - s.z;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq_seed(r2);
        if (CHECK) y0 = (s.g == t.g) ? 0.0 : y0;
        const double ir = rsq_refine(r2, y0);
        const double ir2 = ir * ir;
        const double ir5 = ir * ir2 * ir2;
        const double dqx = s.qx - t.qx, dqy = s.qy - t.qy, dqz = s.qz - t.qz;
        const double qr = fma(dqx, rx, fma(dqy, ry, dqz * rz));
        const double nr = fma(s.nx, rx, fma(s.ny, ry, s.nz * rz));  // n already carries w_j
        const double c = qr * nr * ir5;
        u[0] = fma(c, rx, u[0]);
        u[1] = fma(c, ry, u[1]);
        u[2] = fma(c, rz, u[2]);
    }
};

// Row sums: 6 symmetric accumulators, written as (n,3,3).  Source slots:
// x y z (w n)xyz, g = node index.
struct RowsumP {
    static constexpr int NACC = 6;
    static constexpr int NOUT = 9;
    static constexpr bool kBad = false;
    static constexpr bool kFloatPositions = false;
    __device__ static void target_pos(const PairArgs &a, int64_t i, double *x) { target_xyz(a, i, x); }
    template <class T> __device__ static int target_group(const T &t) { return t.g; }
    typedef TargetBase Target;
    struct SrcR {
        double x, y, z, nx, ny, nz;
        int g;
    };
    typedef double TAcc[1];
    __device__ static void load_target(const PairArgs &a, int64_t i, Target &t) {
        load_target_base(a, i, t, true);
    }
    __device__ static void load_src(const Src80 &s, SrcR &r) {
        r.x = s.v[0]; r.y = s.v[1]; r.z = s.v[2];
        r.nx = s.v[3]; r.ny = s.v[4]; r.nz = s.v[5];
        r.g = s.g;
    }
    __device__ static void zero(TAcc &) {}
    __device__ static void flush(TAcc &, double *) {}
    template <bool CHECK>
    __device__ __forceinline__ static void pair(const Target &t, const SrcR &s, TAcc &, double *u,
                                                int &) {
        const double rx = t.x - s.x, ry = t.y - s.y, rz = t.z - s.z;
        const double r2 = fma(rx, rx, fma(ry, ry, rz * rz));
        double y0 = rsq_seed(r2);
        if (CHECK) y0 = (s.g == t.g) ? 0.0 : y0;
        const double ir = rsq_refine(r2, y0);
        const double ir2 = ir * ir;
        const double ir5 = ir * ir2 * ir2;
        const double c = fma(s.nx, rx, fma(s.ny, ry, s.nz * rz)) * ir5;
        const double cx = c * rx, cy = c * ry, cz = c * rz;
        u[0] = fma(cx, rx, u[0]);
        u[1] = fma(cx, ry, u[1]);
        u[2] = fma(cx, rz, u[2]);
        u[3] = fma(cy, ry, u[3]);
        u[4] = fma(cy, rz, u[4]);
        u[5] = fma(cz, rz, u[5]);
    }
};

template <class P>
__device__ __forceinline__ void write_out(double *dst, const double *u, double scale,
                                          int accumulate = 0) {
    if (P::NOUT == 3) {
        if (accumulate) {
            dst[0] += scale * u[0];
            dst[1] += scale * u[1];
            dst[2] += scale * u[2];
        } else {
            dst[0] = scale * u[0];
            dst[1] = scale * u[1];
            dst[2] = scale * u[2];
        }
    } else {  // symmetric 3x3 from xx xy xz yy yz zz
        dst[0] = scale * u[0]; dst[1] = scale * u[1]; dst[2] = scale * u[2];
        dst[3] = scale * u[1]; dst[4] = scale * u[3]; dst[5] = scale * u[4];
        dst[6] = scale * u[2]; dst[7] = scale * u[4]; dst[8] = scale * u[5];
    }
}

// ----------------------------------------------------------------- engine ----
// Per-tile bounds (TS consecutive packed sources): coordinate box and the
// range of non-negative group ids.  A tile whose box is farther than
// kFastTileMinDist2 from the CTA's target box and whose groups cannot equal
// any target group needs neither the exclusion test nor the r^2 < 1e-24
// test: its pairs run the check-free inner loop.  Only tiles near the CTA's
// own targets (its own fibers, genuinely close neighbours) take the checked
// loop, so results are identical to checking every pair.
struct __align__(16) TileMeta {
    double lo[3], hi[3];
    int gmin, gmax;
    int all_grouped;   // every source of the tile has a group id >= 0
};

template <int TS>
__global__ void tile_meta_kernel(const Src80 *__restrict__ src, int64_t ns,
                                 TileMeta *__restrict__ meta, bool pos_float_hi) {
    __shared__ double red[6][TS / 32];
    __shared__ int gred[2][TS / 32];
    const int64_t j = (int64_t)blockIdx.x * TS + threadIdx.x;
    double v[6];
    int gmn = 0x7fffffff, gmx = (int)0x80000000;
    const int ungrouped = __syncthreads_or(j < ns && src[j].g < 0);
    if (j < ns) {
        const Src80 &q = src[j];
        double x, y, z;
        if (pos_float_hi) {  // FP32c packing: coordinate = hi + lo floats
            const float *f = reinterpret_cast<const float *>(&q);
            x = (double)f[0] + (double)f[3];
            y = (double)f[1] + (double)f[4];
            z = (double)f[2] + (double)f[5];
        } else {
            x = q.v[0]; y = q.v[1]; z = q.v[2];
        }
        v[0] = x; v[1] = y; v[2] = z; v[3] = x; v[4] = y; v[5] = z;
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
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        for (int c = 0; c < 6; ++c) red[c][w] = v[c];
        gred[0][w] = gmn;
        gred[1][w] = gmx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        TileMeta m;
        for (int c = 0; c < 3; ++c) {
            m.lo[c] = red[c][0];
            m.hi[c] = red[3 + c][0];
        }
        m.gmin = gred[0][0];
        m.gmax = gred[1][0];
        m.all_grouped = !ungrouped;
        for (int k = 1; k < TS / 32; ++k) {
            for (int c = 0; c < 3; ++c) {
                m.lo[c] = fmin(m.lo[c], red[c][k]);
                m.hi[c] = fmax(m.hi[c], red[3 + c][k]);
            }
            m.gmin = min(m.gmin, gred[0][k]);
            m.gmax = max(m.gmax, gred[1][k]);
        }
        meta[blockIdx.x] = m;
    }
}

// Tile/box separation below which the checked loop runs: far above
// MIN_SEPARATION^2 = 1e-24, so rounding in r^2 cannot flip a skip decision.
constexpr double kFastTileMinDist2 = 1e-20;

template <class P, int TB, int NT, int TS, int MINB = 1, int UNR = 2>
__global__ void __launch_bounds__(NT, MINB) pair_kernel(PairArgs a,
                                                        const TileMeta *__restrict__ meta) {
    __shared__ __align__(128) Src80 tile[2][TS];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ double tbox[6][NT / 32];
    __shared__ int tgr[2][NT / 32];
    const int tid = threadIdx.x;
    const int64_t tbase = (int64_t)blockIdx.x * (NT * TB);

    typename P::Target tg[TB];
    typename P::TAcc ta[TB];
    double u[TB][P::NACC];
    int nb[TB];
    double bx[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
    int gmn = 0x7fffffff, gmx = (int)0x80000000;
    bool tneg = false;   // some target excludes nothing (group < 0)
#pragma unroll
    for (int k = 0; k < TB; ++k) {
        int64_t i = tbase + k * NT + tid;
        if (i >= a.nt) i = a.nt - 1;  // replicate a real target; results discarded
        P::load_target(a, i, tg[k]);
        P::zero(ta[k]);
#pragma unroll
        for (int c = 0; c < P::NACC; ++c) u[k][c] = 0.0;
        nb[k] = 0;
        double xyz[3];
        P::target_pos(a, i, xyz);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            bx[c] = fmin(bx[c], xyz[c]);
            bx[3 + c] = fmax(bx[3 + c], xyz[c]);
        }
        const int g = P::target_group(tg[k]);
        if (g >= 0) {
            gmn = min(gmn, g);
            gmx = max(gmx, g);
        } else {
            tneg = true;
        }
    }
    // a tile whose sources all share the single group of every target of the
    // CTA is excluded pair by pair: skip it (the reference evaluates and
    // discards those pairs; the sums are identical)
    const bool cta_neg = __syncthreads_or(tneg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            bx[c] = fmin(bx[c], __shfl_xor_sync(0xffffffffu, bx[c], o));
            bx[3 + c] = fmax(bx[3 + c], __shfl_xor_sync(0xffffffffu, bx[3 + c], o));
        }
        gmn = min(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
        gmx = max(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
    }
    if ((tid & 31) == 0) {
        for (int c = 0; c < 6; ++c) tbox[c][tid >> 5] = bx[c];
        tgr[0][tid >> 5] = gmn;
        tgr[1][tid >> 5] = gmx;
    }

    const int64_t j0 = (int64_t)blockIdx.y * a.chunk;
    const int64_t j1 = imin64(a.ns, j0 + a.chunk);
    const int ntiles = j1 > j0 ? (int)((j1 - j0 + TS - 1) / TS) : 0;
    const int64_t tile0 = j0 / TS;  // chunks are TS-aligned

    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // CTA-wide target bounds (identical in every thread)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        bx[c] = tbox[c][0];
        bx[3 + c] = tbox[3 + c][0];
    }
    gmn = tgr[0][0];
    gmx = tgr[1][0];
    for (int w = 1; w < NT / 32; ++w) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            bx[c] = fmin(bx[c], tbox[c][w]);
            bx[3 + c] = fmax(bx[3 + c], tbox[3 + c][w]);
        }
        gmn = min(gmn, tgr[0][w]);
        gmx = max(gmx, tgr[1][w]);
    }

    if (tid == 0 && ntiles > 0) {
        const uint32_t bytes = (uint32_t)(imin64(TS, j1 - j0) * sizeof(Src80));
        mbar_arrive_expect_tx(&full[0], bytes);
        bulk_g2s(tile[0], a.src + j0, bytes, &full[0]);
    }
    for (int t = 0; t < ntiles; ++t) {
        const int s = t & 1;
        // classify the tile while its bytes land
        const TileMeta m = meta[tile0 + t];
        double d2 = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double gap = fmax(0.0, fmax(m.lo[c] - bx[3 + c], bx[c] - m.hi[c]));
            d2 = fma(gap, gap, d2);
        }
        const bool fast = (d2 > kFastTileMinDist2) && (m.gmax < gmn || m.gmin > gmx);
        const bool excluded = !cta_neg && m.all_grouped && m.gmin == m.gmax && gmn == gmx &&
                              m.gmin == gmn;
        mbar_wait(&full[s], (uint32_t)((t >> 1) & 1));
        __syncthreads();  // all threads are done with tile t-1 (buffer s^1)
        if (tid == 0 && t + 1 < ntiles) {
            const int64_t b = j0 + (int64_t)(t + 1) * TS;
            const uint32_t bytes = (uint32_t)(imin64(TS, j1 - b) * sizeof(Src80));
            mbar_arrive_expect_tx(&full[s ^ 1], bytes);
            bulk_g2s(tile[s ^ 1], a.src + b, bytes, &full[s ^ 1]);
        }
        const int cnt = (int)imin64(TS, j1 - (j0 + (int64_t)t * TS));
        const Src80 *ts = tile[s];
        if (excluded) {
            // nothing to add
        } else if (fast && cnt == TS) {
#pragma unroll UNR
            for (int jj = 0; jj < TS; ++jj) {
                typename P::SrcR sr;
                P::load_src(ts[jj], sr);
                FastStep<P, TB>::run(tg, sr, ta, u, nb);
            }
        } else {
            for (int jj = 0; jj < cnt; ++jj) {
                typename P::SrcR sr;
                P::load_src(ts[jj], sr);
#pragma unroll
                for (int k = 0; k < TB; ++k) P::template pair<true>(tg[k], sr, ta[k], u[k], nb[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < TB; ++k) P::flush(ta[k], u[k]);
    }

    int nbad = 0;
#pragma unroll
    for (int k = 0; k < TB; ++k) {
        const int64_t i = tbase + k * NT + tid;
        if (i < a.nt) {
            nbad += nb[k];
            if (a.nsplit == 1) {
                write_out<P>(a.out + (int64_t)P::NOUT * i, u[k], a.pref, a.accumulate);
            } else {
                double *dst = a.partial + ((int64_t)blockIdx.y * a.nt + i) * P::NACC;
#pragma unroll
                for (int c = 0; c < P::NACC; ++c) dst[c] = u[k][c];
            }
        }
    }
    if (P::kBad && a.bad) {
        nbad = warp_sum_int(nbad);
        if ((tid & 31) == 0 && nbad) atomicAdd(a.bad, (unsigned long long)nbad);
    }
}

template <class P>
__global__ void reduce_partials(const double *__restrict__ partial, int nsplit, int64_t nt,
                                double pref, double *__restrict__ out, int accumulate) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nt) return;
    double u[P::NACC];
#pragma unroll
    for (int c = 0; c < P::NACC; ++c) u[c] = 0.0;
    // chunk order as before; the loads of 4 chunks are issued together (the
    // one-load-per-add loop ran latency-bound with only nt threads: 21-45 us
    // for the 1,024 C2 particle targets over 128 chunks)
    const int64_t stride = nt * P::NACC;
    const double *p = partial + i * P::NACC;
    int s = 0;
    for (; s + 4 <= nsplit; s += 4) {
        double v[4][P::NACC];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < P::NACC; ++c) v[k][c] = __ldcs(p + (s + k) * stride + c);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int c = 0; c < P::NACC; ++c) u[c] += v[k][c];
    }
    for (; s < nsplit; ++s)
#pragma unroll
        for (int c = 0; c < P::NACC; ++c) u[c] += __ldcs(p + s * stride + c);
    write_out<P>(out + (int64_t)P::NOUT * i, u, pref, accumulate);
}

// The same chunk-order sums with one thread per output element (NOUT == NACC
// == 3): 3x the threads, and the loads of 8 chunks issued together; few-target
// launches (1,024 C2 particle nodes x 128 chunks) ran latency-bound at one
// load per add per target (21-45 us).  Bit-identical to reduce_partials.
__global__ void reduce_partials3(const double *__restrict__ partial, int nsplit, int64_t nt,
                                 double pref, double *__restrict__ out, int accumulate) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 3 * nt) return;
    const int64_t stride = 3 * nt;
    const double *p = partial + e;
    double u = 0.0;
    int s = 0;
    for (; s + 8 <= nsplit; s += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + (s + k) * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k) u += v[k];
    }
    for (; s < nsplit; ++s) u += __ldcs(p + s * stride);
    out[e] = accumulate ? out[e] + pref * u : pref * u;
}

// ---------------------------------------------------------------- packing ----
// wsrc (nullable) folds the quadrature weight into the strength on the fly:
// f_j <- w_j f_j (system.py:657-658).
__global__ void pack_sbt(const double *__restrict__ src, const int64_t *__restrict__ sgrp,
                         const double *__restrict__ f, const double *__restrict__ dcoef,
                         int64_t ns, Src80 *__restrict__ out,
                         const double *__restrict__ wsrc = nullptr) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ns;
         j += (int64_t)gridDim.x * blockDim.x) {
        Src80 s;
        const double wj = wsrc ? wsrc[j] : 1.0;
        s.v[0] = src[3 * j]; s.v[1] = src[3 * j + 1]; s.v[2] = src[3 * j + 2];
        if (wsrc) {
            s.v[3] = wj * f[3 * j]; s.v[4] = wj * f[3 * j + 1]; s.v[5] = wj * f[3 * j + 2];
        } else {
            s.v[3] = f[3 * j]; s.v[4] = f[3 * j + 1]; s.v[5] = f[3 * j + 2];
        }
        const double c = dcoef ? dcoef[j] : 0.0;
        s.v[6] = c; s.v[7] = 3.0 * c; s.v[8] = 0.0;
        s.g = sgrp ? pack_source_group(sgrp[j]) : -1;
        s.pad = 0;
        out[j] = s;
    }
}

__global__ void pack_sbt_f32c(const double *__restrict__ src, const int64_t *__restrict__ sgrp,
                              const double *__restrict__ f, const double *__restrict__ dcoef,
                              int64_t ns, Src80 *__restrict__ out,
                              const double *__restrict__ wsrc = nullptr) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ns;
         j += (int64_t)gridDim.x * blockDim.x) {
        Src80 s;
        float *p = reinterpret_cast<float *>(&s);
        for (int c = 0; c < 3; ++c) {
            const double x = src[3 * j + c];
            const float h = __double2float_rn(x);
            p[c] = h;
            p[3 + c] = __double2float_rn(x - (double)h);
            p[6 + c] = __double2float_rn(wsrc ? wsrc[j] * f[3 * j + c] : f[3 * j + c]);
        }
        const double c = dcoef ? dcoef[j] : 0.0;
        p[9] = __double2float_rn(c);
        p[10] = __double2float_rn(3.0 * c);
        for (int c2 = 11; c2 < 18; ++c2) p[c2] = 0.f;
        s.g = sgrp ? pack_source_group(sgrp[j]) : -1;
        s.pad = 0;
        out[j] = s;
    }
}

// wsrc (nullable): qw_j <- w_j q_j (system.py:674-679).
__global__ void pack_stresslet(const double *__restrict__ src, const int64_t *__restrict__ sgrp,
                               const double *__restrict__ nrm, const double *__restrict__ qw,
                               int64_t ns, Src80 *__restrict__ out,
                               const double *__restrict__ wsrc = nullptr) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ns;
         j += (int64_t)gridDim.x * blockDim.x) {
        Src80 s;
        for (int c = 0; c < 3; ++c) {
            s.v[c] = src[3 * j + c];
            s.v[3 + c] = nrm[3 * j + c];
            s.v[6 + c] = wsrc ? qw[3 * j + c] * wsrc[j] : qw[3 * j + c];
        }
        s.g = sgrp ? pack_source_group(sgrp[j]) : -1;
        s.pad = 0;
        out[j] = s;
    }
}

// q == nullptr packs for the row sum (slots 6..8 zero).
__global__ void pack_surface_self(const double *__restrict__ nodes, const double *__restrict__ nrm,
                                  const double *__restrict__ w, const double *__restrict__ q,
                                  int64_t n, Src80 *__restrict__ out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        Src80 s;
        for (int c = 0; c < 3; ++c) {
            s.v[c] = nodes[3 * j + c];
            s.v[3 + c] = w[j] * nrm[3 * j + c];
            s.v[6 + c] = q ? q[3 * j + c] : 0.0;
        }
        s.g = (int)j;
        s.pad = 0;
        out[j] = s;
    }
}

// ----------------------------------------------------------------- launch ----
namespace {
// Default launch shape (measured on B200, tools/gpu_sweep.sh): 1 target per
// thread, 128 threads, >= 8 CTAs per SM (64 registers), 4 sources unrolled.
constexpr int kNT = 128;
constexpr int kTB = 1;
constexpr int kMinBlocks = 8;
constexpr int kUnroll = 4;
constexpr int kTS = 128;
constexpr int kTargetsPerCta = kNT * kTB;

// Split factor from (nt, ns) only: aim for >= 16384 (target block x source
// chunk) work units so the last wave is a small fraction of the grid, while
// keeping every chunk >= 4 tiles.
int choose_split(int64_t nt, int64_t ns) {
    const int64_t blocks = (nt + kTargetsPerCta - 1) / kTargetsPerCta;
    static const int min_tiles = [] {   // source tiles per split (tuning knob)
        // 2 (r02 A/B): finer source splits for few-target launches, such as
        // the C2 particle targets x fiber sources sum on the side stream,
        // fill the symmetric kernel's gaps better (C2 matvec + precond
        // 2.02 -> 1.98 ms, C1 step 5.67 -> 5.53 ms, C4 unchanged)
        const char *e = getenv("SF_SPLIT_TILES");
        return e ? atoi(e) : 2;
    }();
    int64_t s = (16384 + blocks - 1) / blocks;
    int64_t max_s = ns / (min_tiles * kTS);
    // small problems: split down to one source tile per CTA if that is what
    // it takes to give every SM two CTAs
    const int64_t fill = (2 * 148 + blocks - 1) / blocks;
    if (max_s < fill) max_s = fill < ns / kTS ? fill : ns / kTS;
    if (s > max_s) s = max_s;
    if (s > 256) s = 256;
    return s < 1 ? 1 : (int)s;
}

int pack_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g > 4096 ? 4096 : (g < 1 ? 1 : g));
}
}  // namespace

int pair_split(int64_t nt, int64_t ns) {
    if (nt <= 0 || ns <= 0) return 0;
    int s = choose_split(nt, ns);
    if (s > 1) {
        int64_t chunk = (ns + s - 1) / s;
        chunk = ((chunk + kTS - 1) / kTS) * kTS;
        s = (int)((ns + chunk - 1) / chunk);
    }
    return s < 1 ? 1 : s;
}

template <class P>
static int launch_pairs(PairArgs a, cudaStream_t st, Workspace &ws) {
    if (a.nt == 0) return 0;
    a.nsplit = choose_split(a.nt, a.ns);
    a.chunk = (a.ns + a.nsplit - 1) / a.nsplit;
    a.chunk = ((a.chunk + kTS - 1) / kTS) * kTS;
    if (a.nsplit > 1) {
        a.nsplit = (int)((a.ns + a.chunk - 1) / a.chunk);
        if (a.nsplit < 1) a.nsplit = 1;
    }
    if (a.nsplit > 1) {
        a.partial = (double *)ws.get(1, sizeof(double) * (size_t)a.nsplit * a.nt * P::NACC, st);
        if (!a.partial) return SF_ENOMEM;
    }
    const int64_t ntiles = (a.ns + kTS - 1) / kTS;
    TileMeta *meta = (TileMeta *)ws.get(2, sizeof(TileMeta) * (size_t)ntiles, st);
    if (!meta) return SF_ENOMEM;
    tile_meta_kernel<kTS><<<(unsigned)ntiles, kTS, 0, st>>>(a.src, a.ns, meta,
                                                           P::kFloatPositions);
    // SF_PAIR_VARIANT (tuning experiments only) picks the launch shape.
    static const int variant = [] {
        const char *e = getenv("SF_PAIR_VARIANT");
        return e ? atoi(e) : 0;
    }();
    const unsigned ny = (unsigned)a.nsplit;
    auto nb = [&](int per) { return (unsigned)((a.nt + per - 1) / per); };
    switch (variant) {
        case 1: pair_kernel<P, 1, 128, kTS, 8, 2><<<dim3(nb(128), ny), 128, 0, st>>>(a, meta); break;
        case 2: pair_kernel<P, 2, 128, kTS, 8, 2><<<dim3(nb(256), ny), 128, 0, st>>>(a, meta); break;
        case 3: pair_kernel<P, 1, 256, kTS, 4, 2><<<dim3(nb(256), ny), 256, 0, st>>>(a, meta); break;
        case 4: pair_kernel<P, 1, 128, kTS, 10, 2><<<dim3(nb(128), ny), 128, 0, st>>>(a, meta); break;
        case 5: pair_kernel<P, 2, 256, kTS, 4, 2><<<dim3(nb(512), ny), 256, 0, st>>>(a, meta); break;
        case 7: pair_kernel<P, 2, 128, kTS, 6, 4><<<dim3(nb(256), ny), 128, 0, st>>>(a, meta); break;
        case 8: pair_kernel<P, 1, 256, kTS, 4, 4><<<dim3(nb(256), ny), 256, 0, st>>>(a, meta); break;
        default:
            pair_kernel<P, kTB, kNT, kTS, kMinBlocks, kUnroll>
                <<<dim3(nb(kTargetsPerCta), ny), kNT, 0, st>>>(a, meta);
    }
    if (a.nsplit > 1) {
        if (P::NOUT == 3 && P::NACC == 3)
            reduce_partials3<<<(unsigned)((3 * a.nt + 127) / 128), 128, 0, st>>>(
                a.partial, a.nsplit, a.nt, a.pref, a.out, a.accumulate);
        else
            reduce_partials<P><<<(unsigned)((a.nt + 255) / 256), 256, 0, st>>>(a.partial, a.nsplit,
                                                                          a.nt, a.pref, a.out,
                                                                          a.accumulate);
    }
    return check_launch("pair_kernel");
}

int pairs_sbt(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
              const int64_t *sgrp, int64_t ns, const double *f, const double *dcoef, double pref,
              int mode, double *out, int64_t *bad, cudaStream_t st, Workspace &ws) {
    return pairs_sbt_weighted(trg, tgrp, nt, src, sgrp, ns, f, nullptr, dcoef, pref, mode, out,
                              bad, st, ws);
}

int pairs_sbt_weighted(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                       const int64_t *sgrp, int64_t ns, const double *f, const double *wsrc,
                       const double *dcoef, double pref, int mode, double *out, int64_t *bad,
                       cudaStream_t st, Workspace &ws, int accumulate) {
    if (bad) {
        if (cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess) return check_launch("memset");
    }
    if (nt == 0) return 0;
    if (ns == 0) {
        if (accumulate) return 0;
        if (cudaMemsetAsync(out, 0, sizeof(double) * 3 * nt, st) != cudaSuccess)
            return check_launch("memset");
        return 0;
    }
    Src80 *packed = (Src80 *)ws.get(0, sizeof(Src80) * (size_t)ns, st);
    if (!packed) return SF_ENOMEM;
    PairArgs a{};
    a.trg = trg; a.tgrp = tgrp; a.nt = nt; a.src = packed; a.ns = ns; a.pref = pref;
    a.out = out; a.bad = (unsigned long long *)bad; a.accumulate = accumulate;
    if (mode == 1) {
        pack_sbt_f32c<<<pack_grid(ns), 256, 0, st>>>(src, sgrp, f, dcoef, ns, packed, wsrc);
        return launch_pairs<SbtF32cP>(a, st, ws);
    }
    pack_sbt<<<pack_grid(ns), 256, 0, st>>>(src, sgrp, f, dcoef, ns, packed, wsrc);
    if (dcoef) return launch_pairs<SbtP<true>>(a, st, ws);
    return launch_pairs<SbtP<false>>(a, st, ws);
}

int pairs_doublet_only(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                       const int64_t *sgrp, int64_t ns, const double *f, double pref, double *out,
                       int64_t *bad, cudaStream_t st, Workspace &ws) {
    if (bad) {
        if (cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess) return check_launch("memset");
    }
    if (nt == 0) return 0;
    if (ns == 0) {
        if (cudaMemsetAsync(out, 0, sizeof(double) * 3 * nt, st) != cudaSuccess)
            return check_launch("memset");
        return 0;
    }
    Src80 *packed = (Src80 *)ws.get(0, sizeof(Src80) * (size_t)ns, st);
    if (!packed) return SF_ENOMEM;
    pack_sbt<<<pack_grid(ns), 256, 0, st>>>(src, sgrp, f, nullptr, ns, packed);
    PairArgs a{};
    a.trg = trg; a.tgrp = tgrp; a.nt = nt; a.src = packed; a.ns = ns; a.pref = pref;
    a.out = out; a.bad = (unsigned long long *)bad;
    return launch_pairs<DoubletP>(a, st, ws);
}

int pairs_stresslet(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                    const int64_t *sgrp, int64_t ns, const double *nrm, const double *qw,
                    double pref, double *out, int64_t *bad, cudaStream_t st, Workspace &ws,
                    const double *wsrc, int accumulate) {
    if (bad) {
        if (cudaMemsetAsync(bad, 0, sizeof(int64_t), st) != cudaSuccess) return check_launch("memset");
    }
    if (nt == 0) return 0;
    if (ns == 0) {
        if (accumulate) return 0;
        if (cudaMemsetAsync(out, 0, sizeof(double) * 3 * nt, st) != cudaSuccess)
            return check_launch("memset");
        return 0;
    }
    Src80 *packed = (Src80 *)ws.get(0, sizeof(Src80) * (size_t)ns, st);
    if (!packed) return SF_ENOMEM;
    pack_stresslet<<<pack_grid(ns), 256, 0, st>>>(src, sgrp, nrm, qw, ns, packed, wsrc);
    PairArgs a{};
    a.trg = trg; a.tgrp = tgrp; a.nt = nt; a.src = packed; a.ns = ns; a.pref = pref;
    a.out = out; a.bad = (unsigned long long *)bad; a.accumulate = accumulate;
    return launch_pairs<StressletP>(a, st, ws);
}

int pairs_dl_subtracted(const double *nodes, const double *nrm, const double *w, const double *q,
                        int64_t n, double pref, double *out, cudaStream_t st, Workspace &ws) {
    if (n == 0) return 0;
    if (use_dl_symmetric(n))
        return pairs_dl_subtracted_symmetric(nodes, nrm, w, q, n, pref, out, st, ws);
    Src80 *packed = (Src80 *)ws.get(0, sizeof(Src80) * (size_t)n, st);
    if (!packed) return SF_ENOMEM;
    pack_surface_self<<<pack_grid(n), 256, 0, st>>>(nodes, nrm, w, q, n, packed);
    PairArgs a{};
    a.trg = nodes; a.tq = q; a.nt = n; a.src = packed; a.ns = n; a.pref = pref; a.out = out;
    return launch_pairs<DlSubP>(a, st, ws);
}

int pairs_rowsum(const double *nodes, const double *nrm, const double *w, int64_t n, double pref,
                 double *out, cudaStream_t st, Workspace &ws) {
    if (n == 0) return 0;
    Src80 *packed = (Src80 *)ws.get(0, sizeof(Src80) * (size_t)n, st);
    if (!packed) return SF_ENOMEM;
    pack_surface_self<<<pack_grid(n), 256, 0, st>>>(nodes, nrm, w, nullptr, n, packed);
    PairArgs a{};
    a.trg = nodes; a.nt = n; a.src = packed; a.ns = n; a.pref = pref; a.out = out;
    return launch_pairs<RowsumP>(a, st, ws);
}

}  // namespace sf
