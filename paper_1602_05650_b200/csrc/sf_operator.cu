// sf_operator.cu — complementary_velocities (system.py:623-709) on the
// device: every family of the HI operator applied to one frozen layout (the
// reference's InteractionCache, system.py:492-562) in a fixed order:
//   1. fiber sources -> all targets: fused Stokeslet + (eps L)^2/2 doublet
//   2. surface sources -> all targets: stresslet (double layer) with q w
//   3. completion flow of every rigid particle's wrench (Stokeslet + rotlet)
//   4. near-field correction maps (block-sparse, CSR by target)
#include <cmath>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <unordered_map>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

// system.py:689-700: u[t] += pref (F/d + (r.F) r/d^3) ; u[t] += pref (L x r)/d^3
// for every target outside the particle's own group.
__global__ void completion_kernel(const double *__restrict__ trg, const int64_t *__restrict__ tgrp,
                                  int64_t nt, const double *__restrict__ centers,
                                  const int64_t *__restrict__ pgrp, int64_t np,
                                  const double *__restrict__ wrench, double pref,
                                  double *__restrict__ u, unsigned long long *bad) {
    int nbad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = trg[3 * i], y = trg[3 * i + 1], z = trg[3 * i + 2];
        const int64_t g = tgrp ? tgrp[i] : -1;
        double ux = u[3 * i], uy = u[3 * i + 1], uz = u[3 * i + 2];
        for (int64_t p = 0; p < np; ++p) {
            if (g == pgrp[p]) continue;
            const double rx = x - centers[3 * p], ry = y - centers[3 * p + 1],
                         rz = z - centers[3 * p + 2];
            const double d = sqrt(rx * rx + ry * ry + rz * rz);
            if (d < 1e-12) {
                ++nbad;
                continue;
            }
            const double *W = wrench + 6 * p;  // F, L
            const double d3 = d * d * d;
            const double rF = (rx * W[0] + ry * W[1] + rz * W[2]) / d3;
            ux += pref * (W[0] / d + rF * rx);
            uy += pref * (W[1] / d + rF * ry);
            uz += pref * (W[2] / d + rF * rz);
            ux += pref * (W[4] * rz - W[5] * ry) / d3;
            uy += pref * (W[5] * rx - W[3] * rz) / d3;
            uz += pref * (W[3] * ry - W[4] * rx) / d3;
        }
        u[3 * i] = ux;
        u[3 * i + 1] = uy;
        u[3 * i + 2] = uz;
    }
    nbad = warp_sum_int(nbad);
    if ((threadIdx.x & 31) == 0 && nbad && bad) atomicAdd(bad, (unsigned long long)nbad);
}

// u += pref * t, contracted to one FMA per entry exactly as the pair
// kernels' accumulating epilogue (write_out) is, so a sum computed with
// scale 1 into t and added here equals the in-kernel accumulation bit for bit.
__global__ void fma_add_kernel(double *__restrict__ u, const double *__restrict__ t, double pref,
                               int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        u[i] = fma(pref, t[i], u[i]);
}

__global__ void add_counter_kernel(int64_t *dst, const int64_t *src) { dst[0] += src[0]; }

int add_counter(int64_t *dst, const int64_t *src, cudaStream_t st) {
    add_counter_kernel<<<1, 1, 0, st>>>(dst, src);
    return check_launch("add_counter_kernel");
}

// A side stream per caller stream (the last stream of the caller's SidePool;
// the symmetric fiber kernel's waves use the others), forked from and joined
// back into it with events, so the small non-fiber-target x fiber-source sum
// (rows [0, off)) overlaps the symmetric fiber block (rows [off, nt)): the two
// write disjoint rows, so the result is bit-identical to running them in
// order.  SF_OVERLAP=0 serialises (A/B measurements; read once).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

static bool side_for(cudaStream_t st, SideStream *out) {
    static const bool enabled = [] {
        const char *e = getenv("SF_OVERLAP");
        return !(e && atoi(e) == 0);
    }();
    if (!enabled) return false;
    SidePool *p = side_pool_for(st);
    if (!p) return false;
    out->s = p->s[SidePool::kStreams - 1];
    out->fork = p->fork;
    out->join = p->done[SidePool::kStreams];
    return true;
}

}  // namespace sf

using namespace sf;

extern "C" int sf_hi_apply(const sf_hi_layout *L, const double *f, const double *q,
                           const double *wrench, const double *near_x, double *u, int64_t *bad,
                           void *stream) {
    if (!L) return set_error(SF_EINVAL, "null layout");
    if (L->nt < 0 || L->nfs < 0 || L->nss < 0 || L->np < 0 || L->near_nrows < 0)
        return set_error(SF_EINVAL, "negative size");
    if (L->nt > 0 && (!L->trg || !u)) return set_error(SF_EINVAL, "null target/output pointer");
    if (L->nfs > 0 && (!L->fsrc || !L->fw || !f)) return set_error(SF_EINVAL, "null fiber data");
    if (L->nss > 0 && (!L->ssrc || !L->snrm || !L->sw || !q))
        return set_error(SF_EINVAL, "null surface data");
    if (L->np > 0 && (!L->pcenter || !L->pgrp || !wrench))
        return set_error(SF_EINVAL, "null particle data");
    if (L->near_nrows > 0 && !near_x) return set_error(SF_EINVAL, "near map without x vector");
    if (!(L->mu > 0)) return set_error(SF_EINVAL, "viscosity must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = workspace_for(st);
    int64_t *bad_f = bad, *bad_s = bad ? bad + 1 : nullptr;
    if (bad && cudaMemsetAsync(bad, 0, 3 * sizeof(int64_t), st) != cudaSuccess)
        return check_launch("memset");
    if (L->nt == 0) return SF_OK;
    const double pref = 1.0 / (8.0 * M_PI * L->mu);
    int rc;
    const int64_t off = L->fiber_target_off;
    double *stress_tmp = nullptr;  // surface-source sum computed on the side stream
    const bool sym = L->nfs > 0 && off >= 0 && off + L->nfs == L->nt &&
                     use_symmetric(L->mode, L->nfs);
    // Surface targets are exactly the surface sources (whole system): the
    // fiber <-> surface pairs then run once per pair (sf_cross.cu).
    const bool cross = sym && L->nss > 0 && L->nss == off && use_cross(L->nfs, L->nss);
    if (cross) {
        // surface targets <- surface sources (writes rows [0, off)); kept in
        // order: overlapping it with the symmetric block measured 2-10 %
        // slower at C4 (the two FP64-bound sweeps contend, and the sym
        // kernel's pair-count-balanced tasks lose their balance)
        rc = pairs_stresslet(L->trg, L->tgrp, off, L->ssrc, L->sgrp, L->nss, L->snrm, q,
                             -3.0 / (4.0 * M_PI * L->mu), u, bad_s, st, ws, L->sw, 0);
        if (rc) return rc;
        // fiber targets <- fiber sources, symmetrically (writes rows [off, nt))
        int64_t *bad_sym = nullptr;
        if (bad) {
            bad_sym = (int64_t *)ws.get(6, sizeof(int64_t), st);
            if (!bad_sym) return SF_ENOMEM;
        }
        rc = pairs_sbt_symmetric(L->fsrc, L->fgrp, L->nfs, L->fiber_group_size, f, L->fw,
                                 L->fdcoef, pref, u + 3 * off, bad_sym, 0, st, ws, L->mode);
        if (rc) return rc;
        if (bad) {
            rc = add_counter(bad_f, bad_sym, st);
            if (rc) return rc;
        }
        // fiber targets <- surface sources and surface targets <- fiber sources
        rc = pairs_cross(L->fsrc, f, L->fw, L->fdcoef, L->nfs, L->ssrc, q, L->sw, L->snrm, L->nss,
                         -3.0 / (4.0 * M_PI * L->mu), pref, u + 3 * off, 1, u, 1, bad_s, bad_f,
                         st, ws);
        if (rc) return rc;
    } else if (sym) {
        int64_t *bad_sym = nullptr;
        if (bad) {
            bad_sym = (int64_t *)ws.get(6, sizeof(int64_t), st);
            if (!bad_sym) return SF_ENOMEM;
        }
        // non-fiber targets against fiber sources and every target against
        // the surface sources (on the side stream when there is one),
        // concurrently with the fiber block done symmetrically.  The side
        // work is queued BEFORE the symmetric sum: its first kernel runs
        // beside the task kernel's first blocks and the rest fills the task
        // kernel's last-wave tail.  Forking it after the packing kernels at
        // the highest stream priority (SF_SIDE_FIRST=1) overlaps all of it
        // with the task kernel instead, which measured slower at C2 (2.34 vs
        // 2.28 ms per Arnoldi step): both are FP64-bound, so the task kernel
        // stretches by the side work, and the small side kernels wait ~100 us
        // each for a slot as the long task blocks retire.
        SideStream side_s;
        SideStream *side = ((off > 0 || L->nss > 0) && side_for(st, &side_s)) ? &side_s : nullptr;
        bool forked = false;
        std::function<int()> side_work = [&]() -> int {
            cudaStream_t rs = st;
            if (side) {
                if (cudaEventRecord(side->fork, st) != cudaSuccess ||
                    cudaStreamWaitEvent(side->s, side->fork, 0) != cudaSuccess)
                    return check_launch("side stream fork");
                forked = true;
                rs = side->s;
            }
            Workspace &rws = side ? workspace_for(rs) : ws;
            int r = off > 0 ? pairs_sbt_weighted(L->trg, L->tgrp, off, L->fsrc, L->fgrp, L->nfs, f,
                                                 L->fw, L->fdcoef, pref, SF_MODE_FP64, u, bad_f, rs,
                                                 rws, 0)
                            : SF_OK;
            if (!r && side && L->nss > 0) {
                // the stresslet sum unscaled into a side buffer, added after the join
                stress_tmp = (double *)rws.get(11, sizeof(double) * 3 * (size_t)L->nt, rs);
                r = stress_tmp ? pairs_stresslet(L->trg, L->tgrp, L->nt, L->ssrc, L->sgrp, L->nss,
                                                 L->snrm, q, 1.0, stress_tmp, bad_s, rs, rws,
                                                 L->sw, 0)
                               : SF_ENOMEM;
            }
            if (side && cudaEventRecord(side->join, side->s) != cudaSuccess && !r)
                r = check_launch("side stream join");
            return r;
        };
        static const bool side_first = [] {
            const char *e = getenv("SF_SIDE_FIRST");
            return e && atoi(e) == 1;
        }();
        if (side && side_first) {
            rc = pairs_sbt_symmetric(L->fsrc, L->fgrp, L->nfs, L->fiber_group_size, f, L->fw,
                                     L->fdcoef, pref, u + 3 * off, bad_sym, 0, st, ws, L->mode,
                                     &side_work);
        } else {
            rc = (off > 0 || side) ? side_work() : SF_OK;
            if (!rc)
                rc = pairs_sbt_symmetric(L->fsrc, L->fgrp, L->nfs, L->fiber_group_size, f, L->fw,
                                         L->fdcoef, pref, u + 3 * off, bad_sym, 0, st, ws, L->mode);
        }
        // join before anything else touches rows [0, off) or the counters
        if (forked && cudaStreamWaitEvent(st, side->join, 0) != cudaSuccess && !rc)
            rc = check_launch("side stream wait");
        if (rc) return rc;
        if (bad) {
            rc = add_counter(bad_f, bad_sym, st);
            if (rc) return rc;
        }
    } else if (L->nfs > 0) {
        rc = pairs_sbt_weighted(L->trg, L->tgrp, L->nt, L->fsrc, L->fgrp, L->nfs, f, L->fw,
                                L->fdcoef, pref, L->mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64,
                                u, bad_f, st, ws, 0);
        if (rc) return rc;
    } else if (cudaMemsetAsync(u, 0, sizeof(double) * 3 * L->nt, st) != cudaSuccess) {
        return check_launch("memset");
    }
    if (stress_tmp) {
        const double pref_dl = -3.0 / (4.0 * M_PI * L->mu);
        int64_t n = 3 * L->nt, blocks = (n + 255) / 256;
        if (blocks > 4096) blocks = 4096;
        fma_add_kernel<<<(unsigned)blocks, 256, 0, st>>>(u, stress_tmp, pref_dl, n);
        rc = check_launch("fma_add_kernel");
        if (rc) return rc;
    } else if (L->nss > 0 && !cross) {
        rc = pairs_stresslet(L->trg, L->tgrp, L->nt, L->ssrc, L->sgrp, L->nss, L->snrm, q,
                             -3.0 / (4.0 * M_PI * L->mu), u, bad_s, st, ws, L->sw, 1);
        if (rc) return rc;
    }
    if (L->np > 0) {
        int64_t blocks = (L->nt + 255) / 256;
        if (blocks > 4096) blocks = 4096;
        completion_kernel<<<(unsigned)blocks, 256, 0, st>>>(
            L->trg, L->tgrp, L->nt, L->pcenter, L->pgrp, L->np, wrench, pref, u,
            bad ? (unsigned long long *)(bad + 2) : nullptr);
        rc = check_launch("completion_kernel");
        if (rc) return rc;
    }
    if (L->near_nrows > 0) {
        rc = near_apply(L->near_row_ptr, L->near_rows, L->near_nrows, L->near_w_off,
                        L->near_x_off, L->near_x_len, L->near_W, near_x, u, st);
        if (rc) return rc;
    }
    return SF_OK;
}
