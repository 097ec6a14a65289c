/*
 * sf_b200.h — C ABI of the B200-native hydrodynamic-interaction (HI) operator
 * for the slender-fiber method of arXiv 1602.05650 (reference package
 * `slenderflow`, /root/reference/pkg/src/slenderflow).
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes; no torch or C++ types;
 *   - arrays are C-contiguous: points/vectors (N,3) float64 AoS, group ids
 *     int64 (-1 = no exclusion, kernels.py:337-339), matrices row-major;
 *   - `sf_*` entry points take DEVICE pointers and a cudaStream_t passed as
 *     `void *stream` (NULL = legacy default stream); they allocate nothing,
 *     never synchronise, and return SF_OK (0) or an error code;
 *   - `sf_host_*` entry points take HOST pointers, exactly the arrays the
 *     reference passes to its numba kernels, copy in, run, copy out and
 *     synchronise (the drop-in a ctypes/cffi binding of kernels.py calls);
 *   - `bad` outputs count target/source pairs closer than MIN_SEPARATION
 *     that were skipped (kernels.py:99-101); like the reference the kernels
 *     never raise — callers raise SingularEvaluationError when bad > 0;
 *   - every per-target sum runs over sources in one fixed order, so results
 *     are bitwise reproducible run to run and independent of grid size.
 */
#ifndef SF_B200_H
#define SF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SF_OK = 0,
    SF_EINVAL = 1,  /* bad argument (negative size, NULL pointer with n > 0) */
    SF_ECUDA = 2,   /* CUDA runtime error; see sf_last_error() */
    SF_ENOMEM = 3,  /* device allocation failed (host entry points only) */
    SF_ENODEV = 4   /* no CUDA device */
};

/* Arithmetic mode of the pair kernels. */
enum {
    SF_MODE_FP64 = 0,        /* FP64 compute and accumulation; where targets == sources
                                (the fiber x fiber block, >= 8192 points) each pair's
                                geometry is evaluated once for both directions */
    SF_MODE_FP32C = 1,       /* FP32 pair arithmetic, FP64 accumulation per tile / slab
                                (symmetric where SF_MODE_FP64 would be) */
    SF_MODE_FP64_DIRECT = 2  /* FP64, every target summed over sources in index
                                order (the reference's loop order) */
};

int sf_abi_version(void);
const char *sf_last_error(void);
int sf_device_sm_count(void);

/* ---------------------------------------------------------------------------
 * Pair sums.  Device pointers.  `bad` is a device int64 that the call
 * OVERWRITES with the skipped-pair count (pass NULL to ignore).
 * ------------------------------------------------------------------------- */

/* Replaces kernels.stokeslet_sum (kernels.py:72-111), reached through
 * DirectSummation.stokeslet (system.py:93-105):
 *   out_i = pref * sum_{j: g_j != g_i, r2 >= 1e-24} [f_j/r + (r.f_j) r/r^3]. */
int sf_stokeslet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                     const double *src, const int64_t *sgrp, int64_t ns,
                     const double *f, double pref, double *out, int64_t *bad,
                     void *stream);

/* Replaces kernels.doublet_sum (kernels.py:114-145):
 *   out_i = pref * sum [f_j/r^3 - 3 (r.f_j) r/r^5]. */
int sf_doublet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                   const double *src, const int64_t *sgrp, int64_t ns,
                   const double *f, double pref, double *out, int64_t *bad,
                   void *stream);

/* Fused slender-body pair sum: the Stokeslet sum plus the source-doublet sum
 * in ONE pass (system.py:656-671 issue two passes over the same pairs):
 *   out_i = pref * sum_j [ f_j/r + (r.f_j) r/r^3
 *                        + c_j (f_j/r^3 - 3 (r.f_j) r/r^5) ]
 * f_j are the quadrature-weighted strengths (system.py:657-658) and
 * c_j = (eps_l L_l)^2/2 of the source's fiber (system.py:542, 662-664);
 * dcoef == NULL means c_j = 0 (Stokeslet only).  mode: SF_MODE_*. */
int sf_sbt_pair(const double *trg, const int64_t *tgrp, int64_t nt,
                const double *src, const int64_t *sgrp, int64_t ns,
                const double *f, const double *dcoef, double pref, int mode,
                double *out, int64_t *bad, void *stream);

/* Replaces kernels.stresslet_sum (kernels.py:177-213), pref = -3/(4 pi mu),
 * qw = density times quadrature weight (system.py:673-687, body.py:237-251). */
int sf_stresslet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                     const double *src, const int64_t *sgrp, int64_t ns,
                     const double *nrm, const double *qw, double pref,
                     double *out, int64_t *bad, void *stream);

/* Replaces kernels.stresslet_sum_subtracted (kernels.py:216-249), reached
 * through body.double_layer_onsurface (body.py:254-262). */
int sf_stresslet_sum_subtracted(const double *nodes, const double *nrm,
                                const double *w, const double *q, int64_t n,
                                double pref, double *out, void *stream);
/* Rank `rank` of `world`'s share of the symmetric subtracted double layer
 * (unit-pair tasks split by cost, as sf_sbt_symmetric_partial): out (n,3)
 * receives this rank's contribution to every node; summing over ranks gives
 * sf_stresslet_sum_subtracted. */
int sf_stresslet_sum_subtracted_partial(const double *nodes, const double *nrm, const double *w,
                                        const double *q, int64_t n, double pref, int rank,
                                        int world, double *out, void *stream);

/* Replaces kernels.stresslet_rowsum (kernels.py:252-281); out is (n,3,3). */
int sf_stresslet_rowsum(const double *nodes, const double *nrm, const double *w,
                        int64_t n, double pref, double *out, void *stream);

/* ---------------------------------------------------------------------------
 * Fiber self terms (batched over nf fibers of n nodes; fiber-major arrays).
 * ------------------------------------------------------------------------- */

/* Replaces kernels.kdelta_matrix (kernels.py:284-334) called once per fiber
 * by Fiber.kdelta_matrix (fiber.py:213-222).  X,tang (nf,n,3); s,s_alpha
 * (nf,n); w (n) Clenshaw-Curtis weights shared by all fibers; delta (nf);
 * K (nf,3n,3n) fully overwritten. */
int sf_kdelta_build_batched(const double *X, const double *s,
                            const double *s_alpha, const double *tang,
                            const double *w, int64_t nf, int64_t n,
                            const double *delta, double pref, double *K,
                            void *stream);

/* u = M f + K f (+ u if accumulate): local_mobility_apply (fiber.py:244-250)
 * plus nonlocal_Kdelta_apply (fiber.py:253-258) for every fiber.
 * c_log (nf) = -ln(eps^2 e)/(8 pi mu), c_two = 2/(8 pi mu).  K may be null
 * (local mobility only); c_log = c_two = 0 gives K f alone. */
int sf_self_apply_batched(const double *K, const double *tang,
                          const double *c_log, double c_two, const double *f,
                          int64_t nf, int64_t n, int accumulate, double *u,
                          void *stream);

/* Per-fiber geometry (spectral.arclength_map, spectral.py:139-154, and
 * Fiber.refresh_geometry, fiber.py:133-147): from centrelines X (nf,n,3),
 * the Chebyshev differentiation matrix D (n,n), the arclength integration
 * matrix S (n,n) and Clenshaw-Curtis weights wcc (n), writes s, s_alpha,
 * node weights wcc*s_alpha (fiber.py:172-174) (nf,n), tangents (nf,n,3),
 * L (nf) and, when delta_ratio > 0, delta = delta_ratio * L (fiber.py:144).
 * *degenerate (device int, nullable) counts nodes with s_alpha <= 1e-12. */
int sf_fiber_geometry_batched(const double *X, int64_t nf, int64_t n, const double *D,
                              const double *S, const double *wcc, double delta_ratio,
                              double *s, double *s_alpha, double *tang, double *wnode,
                              double *L, double *delta, int *degenerate, void *stream);

/* The fiber part of the HI operator in one call (system.py:656-671 + 702-707,
 * fiber.py:244-258), for the target fibers [t_fiber0, t_fiber0 + t_nfibers)
 * against ALL nf fibers as sources (the target-block shard of a multi-GPU
 * run; t_fiber0 = 0, t_nfibers = nf on one GPU).  With f (nf*n,3) force
 * densities of every fiber:
 *   out_nl   (t_nfibers*n,3) = Stokeslet + doublet sum over other fibers'
 *              nodes of the strengths wnode_j f_j, plus the near corrections
 *              of the CSR map (rows are shard-local target indices; its x
 *              vector is the global f);
 *   out_self (t_nfibers*n,3) = M f + K f of the target fibers (skipped when
 *              out_self == NULL); K holds the target fibers' matrices.
 * dcoef (nf*n) or NULL; near_nrows == 0 disables the near map. */
int sf_fiber_hi_apply(const double *X, const int64_t *grp, int64_t nf, int64_t n,
                      int64_t t_fiber0, int64_t t_nfibers, const double *wnode,
                      const double *dcoef, double pref, int mode, const double *K,
                      const double *tang, const double *c_log, double c_two,
                      const int64_t *near_row_ptr, const int64_t *near_rows,
                      int64_t near_nrows, const int64_t *near_w_off,
                      const int64_t *near_x_off, const int64_t *near_x_len,
                      const double *near_W, const double *f, double *out_nl,
                      double *out_self, int64_t *bad, void *stream);

/* Symmetric fiber x fiber sum, multi-GPU form: rank `rank` of `world`
 * evaluates its contiguous share of the unit-pair tasks (both directions) and
 * writes its contribution to EVERY point into out (N,3); summing out over
 * ranks (NCCL reduce-scatter to the target blocks) gives the Stokeslet +
 * doublet sum.  world = 1 equals the single-GPU symmetric path.  bad counts
 * this rank's skipped ordered pairs. */
int sf_sbt_symmetric_partial(const double *X, const int64_t *grp, int64_t N,
                             int64_t group_size, const double *f, const double *w,
                             const double *dcoef, double pref, int mode, int rank, int world,
                             double *out, int64_t *bad, void *stream);

/* The same sum over an explicit contiguous range [t0, t0 + ntasks) of the
 * sf_sym_task_count(N, group_size, mode) unit-pair tasks (row-major
 * {g <= h}): a rank's share when the split is chosen by the caller, e.g. by
 * modelled cost (sf_sym_task_costs).  Any partition of the tasks into ranges
 * sums to the full symmetric result. */
int sf_sbt_symmetric_tasks(const double *X, const int64_t *grp, int64_t N,
                           int64_t group_size, const double *f, const double *w,
                           const double *dcoef, double pref, int mode, int64_t t0,
                           int64_t ntasks, double *out, int64_t *bad, void *stream);
int64_t sf_sym_task_count(int64_t N, int64_t group_size, int mode);
/* Points per unit of the symmetric evaluation (units align to fibers). */
int64_t sf_sym_unit_size(int64_t N, int64_t group_size, int mode);
/* Modelled cost (device array, one double per task) of every unit-pair task
 * of the symmetric evaluation of positions X / groups grp: the task kernel's
 * slab-pair decisions replayed, a check-free cell costing 1, a checked cell
 * c_checked and a diagonal-task cell c_diag (geometry only; no forces). */
int sf_sym_task_costs(const double *X, const int64_t *grp, int64_t N, int64_t group_size,
                      int mode, double c_checked, double c_diag, double *cost, void *stream);
/* Non-excluded ordered pair interactions and kernel launches of one
 * sf_sbt_symmetric_tasks call over [t0, t0 + count) (host functions). */
int64_t sf_sym_range_pairs(int64_t N, int64_t group_size, int mode, int64_t t0, int64_t count);
int64_t sf_sym_range_launch_count(int64_t N, int64_t group_size, int mode, int64_t t0,
                                  int64_t count);

/* Source-split factor the pair kernels use for nt targets x ns sources (a
 * pure function of the sizes; each target's sum is split into this many
 * ordered chunks).  Used to count kernel launches. */
int sf_pair_split(int64_t nt, int64_t ns);

/* Non-excluded ordered pair interactions evaluated by rank `rank` of `world`
 * in sf_sbt_symmetric_partial (FP64 mode; the FP32c task split uses smaller
 * units) for N points in groups of group_size (the algorithmic work of that
 * launch; host function, no device access). */
int64_t sf_sym_shard_pairs(int64_t N, int64_t group_size, int rank, int world);

/* Kernels one symmetric fiber-pair evaluation launches for rank `rank` of
 * `world` (pack, slab metas, one task kernel and one ordered reduce per wave
 * of task rows, final scale); host function, no device access. */
int64_t sf_sym_launch_count(int64_t N, int64_t group_size, int mode, int rank, int world);

/* Tuning: partial-sum budget (bytes) of one wave of the symmetric fiber-pair
 * evaluation and the number of wave buffers / streams (<= 3); 0 restores the
 * defaults (SF_SYM_WAVE_MB, SF_SYM_STREAMS, else 192 MB and 2).  The results
 * are bitwise independent of both.  Not thread safe against running calls. */
int sf_sym_set_waves(int64_t bytes, int streams);

/* Device scratch currently held by the library's per-stream workspaces, in
 * bytes (all devices and streams of this process). */
int64_t sf_workspace_bytes(void);

/* Synchronise every device the library used and free all its per-stream
 * workspaces (they regrow on the next call).  Not safe against running calls
 * on other host threads. */
int sf_workspace_release(void);

/* ---------------------------------------------------------------------------
 * complementary_velocities (system.py:623-709) on one frozen layout.
 * ------------------------------------------------------------------------- */

/* The reference's InteractionCache (system.py:492-562) as device arrays.
 * Targets: every constituent's nodes stacked [particles | periphery | fibers]
 * with group ids (fiber m -> m, particle i -> nf + i, periphery -> nf + np).
 * Fiber sources carry node weights w s_alpha and doublet coefficients
 * (eps L)^2/2; surface sources carry normals, quadrature weights and their
 * surface's group id; particles carry centres and group ids.  The near map
 * is CSR by target row; its x vector is [fiber forces | surface densities]
 * flattened (x_off / x_len index into it). */
typedef struct {
    const double *trg;       /* (nt,3) */
    const int64_t *tgrp;     /* (nt) */
    int64_t nt;
    const double *fsrc;      /* (nfs,3) fiber nodes */
    const int64_t *fgrp;     /* (nfs) */
    const double *fw;        /* (nfs) w * s_alpha */
    const double *fdcoef;    /* (nfs) doublet coefficient or NULL (include_doublet=False) */
    int64_t nfs;
    const double *ssrc;      /* (nss,3) surface nodes */
    const double *snrm;      /* (nss,3) */
    const double *sw;        /* (nss) quadrature weights */
    const int64_t *sgrp;     /* (nss) */
    int64_t nss;
    const double *pcenter;   /* (np,3) */
    const int64_t *pgrp;     /* (np) */
    int64_t np;
    const int64_t *near_row_ptr, *near_rows, *near_w_off, *near_x_off, *near_x_len;
    int64_t near_nrows;
    const double *near_W;
    double mu;
    int mode;                /* SF_MODE_* for the fiber pair sum */
    int64_t fiber_target_off; /* targets [off, off+nfs) ARE the fiber sources
                                 (same points, order, groups), or -1 */
    int64_t fiber_group_size; /* nodes per fiber (unit alignment), 0 if unknown */
} sf_hi_layout;

/* u (nt,3) = complementary velocities for fiber force densities f (nfs,3),
 * surface densities q (nss,3) and particle wrenches (np,6: F then L).
 * bad (device int64[3], nullable) receives the skipped-pair counts of the
 * fiber, surface and completion families (system.py:668-670, 684-686, 697). */
int sf_hi_apply(const sf_hi_layout *layout, const double *f, const double *q,
                const double *wrench, const double *near_x, double *u, int64_t *bad,
                void *stream);

/* ---------------------------------------------------------------------------
 * Implicit step (solver.py): block rows, self blocks, preconditioner, Krylov.
 * Unknown vector layout (StepLayout, solver.py:67-110):
 *   [per particle U(3) omega(3) q1(3Np) | periphery q0(3N0) | per fiber X(3n) T(n)]
 * ------------------------------------------------------------------------- */

/* Frozen per-step fiber data (the reference's Fiber objects after
 * refresh_geometry, batched).  bc_kind (nf,2) [plus, minus]: 0 free,
 * 1 prescribedForceTorque, 2 hingedToSurface, 3 clampedToBody; bc_par
 * (nf,2,12): force(3) torque(3) attachment(3) stiffness has_tangent pad;
 * bc_body (nf): body of a clamped minus end or -1. */
typedef struct {
    int64_t nf, n;
    const double *D;         /* (n,n) Chebyshev differentiation in alpha */
    const double *nodes;     /* (n) alpha nodes */
    const double *Dpow;      /* (nf,4,n,n) Ds, Ds2, Ds3, Ds4 */
    const double *X;         /* (nf,n,3) frozen centrelines */
    const double *tang;      /* (nf,n,3) */
    const double *s_alpha;   /* (nf,n) */
    const double *L, *Ldot, *E, *c_log;  /* (nf) */
    double c_two;
    const double *K;         /* (nf,3n,3n) K_delta */
    const double *f_ext;     /* (nf,n,3) or NULL */
    const int *bc_kind;
    const double *bc_par;
    const int *bc_body;
    int64_t np;
    const double *pcenter;   /* (np,3) */
    const int64_t *p_uoff;   /* (np) offset of U in the unknown vector (omega at +3) */
    int64_t fib_off;         /* offset of fiber 0's block */
    double dt, mu;
    /* Mixed Chebyshev orders (one sf_fiber_sys per order class): per-fiber
     * offset of the unknown block [X T] (else fib_off + 4 n m) and of the
     * fiber's first point in the point-ordered force / u_bar arrays (else
     * n m).  Both NULL for a uniform system. */
    const int64_t *u_off;
    const int64_t *pt_off;
} sf_fiber_sys;

/* Ds..Ds4 per fiber (fiber.py:140-143). */
int sf_fiber_dpow(const double *D, const double *s_alpha, int64_t nf, int64_t n, double *Dpow,
                  void *stream);
/* f (nf,n,3) = elastic force of the candidate in u (+ f_ext if constants)
 * (solver.py:313-318, fiber.py:237-241). */
int sf_fiber_forces(const sf_fiber_sys *S, const double *u, int constants, double *f,
                    void *stream);
/* Per-particle wrench (np,6) from clamped fibers (system.py:308-329) + ext
 * (np,6) if constants (solver.py:296-305); work (nf,6) scratch. */
int sf_particle_wrenches(const sf_fiber_sys *S, const double *u, const double *ext,
                         int constants, double *work, double *wout, void *stream);
/* Fiber residual rows into out (solver.py:137-184, fiber.py:375-441); ubar
 * (nf*n,3) complementary velocity at the fiber nodes or NULL.  fpre
 * (optional, point order): the force densities sf_fiber_forces already
 * computed from the same u and constants; the rows then read them instead
 * of re-applying D_s^4 and D_s (bit-identical: same arithmetic).  Ignored
 * when constants are on and S has external forces (the clamped-end rows
 * need the elastic part alone). */
int sf_fiber_rows(const sf_fiber_sys *S, const double *u, const double *fpre, const double *ubar,
                  int constants, double *out, void *stream);
/* Dense 4n x 4n self blocks (solver.py:250-294) into A (nf,4n,4n). */
int sf_fiber_self_blocks(const sf_fiber_sys *S, double *A, void *stream);
/* In-place equilibrated LU with partial pivoting of nb m x m blocks
 * (solver.py:386-404), factors left column-major; r, c (nb,m) scalings;
 * piv (nb,m) 0-based; info (nb): 0 ok, 1 non-finite, 2 zero row, 3 zero pivot. */
int sf_block_lu(double *A, int64_t nb, int64_t m, double *r, double *c, int *piv, int *info,
                void *stream);
/* x = Preconditioner.apply(v) (solver.py:425-429): x[:ndiag] = v/diag; each
 * fiber block b at off0 + m b solved with its equilibrated LU. */
int sf_precond_apply(const double *LU, const double *r, const double *c, const int *piv,
                     int64_t nb, int64_t m, int64_t off0, const double *diag, int64_t ndiag,
                     const double *v, double *x, void *stream);
/* Block solves only, for fibers whose unknown blocks start at boff[b]
 * (mixed-order systems: one call per order class). */
int sf_block_solve(const double *LU, const double *r, const double *c, const int *piv, int64_t nb,
                   int64_t m, const int64_t *boff, const double *v, double *x, void *stream);
/* Surface rows (solver.py:332-355).  kind 0 (particle): rows hold DL_on +
 * wrench flow on entry; adds u_bar, subtracts U + omega x arm; out_uom gets
 * U - <q>/mu, omega - <arm x q>/mu.  kind 1 (periphery): rows hold DL_on on
 * entry; adds q/mu + n flux/(mu area) + u_bar.  work >= 6 doubles. */
int sf_surface_rows(int kind, const double *nodes, const double *nrm, const double *w, int64_t n,
                    const double *center, double area, const double *q, const double *ubar,
                    const double *Uom, double mu, double *work, double *rows, double *out_uom,
                    void *stream);
/* u += Stokeslet + rotlet of wrench (F,L) at center (solver.py:125-134). */
int sf_wrench_flow(const double *trg, int64_t nt, const double *center, const double *wrench,
                   double mu, double *u, void *stream);
/* Krylov vector kernels (deterministic order): out = x.y (sqrt_mode: sqrt);
 * work >= 296 doubles.  y += sgn*(*a) x (mode 0) or y = x / (*a) (mode 2);
 * x += sum_j coef[j] V[j*ld : j*ld+n]. */
int sf_dot(const double *x, const double *y, int64_t n, double *work, double *out, int sqrt_mode,
           void *stream);
int sf_axpy_dev(const double *a, double sgn, int mode, const double *x, double *y, int64_t n,
                void *stream);
int sf_combine(const double *V, int64_t ld, int k, const double *coef, double *x, int64_t n,
               void *stream);
/* One Arnoldi step's modified Gram-Schmidt (solver.py:472-486) in one
 * cooperative launch: hcol[R+1] = |w|; for j <= k: hcol[j] = V_j.w,
 * w -= hcol[j] V_j; hcol[k+1] = |w|; V_{k+1} = w / hcol[k+1].  Bitwise equal
 * to the sf_dot / sf_axpy_dev sequence.  V rows of length ld (R+1 rows,
 * k+1 <= R); work >= 4*296 doubles. */
int sf_gmres_mgs(double *V, int64_t ld, int k, double *w, int64_t n, double *hcol, int R,
                 double *work, void *stream);

/* GMRES Hessenberg / Givens bookkeeping on the device (solver.py:444-516),
 * so the host needs one small status record per Arnoldi step instead of the
 * Hessenberg column.  gs: sf_gmres_state_doubles(R, I) doubles of device
 * state (H, cs, sn, g, y, scalars, residual history; see sf_gmres.cu).
 * sf_gmres_reset: start a solve (iterations = 0).  sf_gmres_cycle: start a
 * cycle, g = beta e_0 and V0 = r / beta (beta a device scalar).
 * sf_gmres_givens: step k of the cycle from hcol (sf_gmres_mgs output):
 * previous rotations, new rotation, g, relative residual |g_{k+1}|/beta0
 * into the history, done = converged | breakdown (|w_orth| <= 1e-12 |w|) |
 * cycle full | iteration cap; a no-op once done (speculative steps);
 * status (optional, 4 doubles) = [done, iterations, rel, k].
 * sf_gmres_update: x += V_k^T triu(H_k)^-1 g_k for the k steps taken. */
int64_t sf_gmres_state_doubles(int R, int max_iterations);
int sf_gmres_reset(double *gs, int R, int max_iterations, double beta0, double tol,
                   void *stream);
int sf_gmres_cycle(double *gs, int R, const double *beta, const double *r, double *V0, int64_t n,
                   void *stream);
int sf_gmres_givens(const double *hcol, double *gs, int R, int k, double *status, void *stream);
/* The same two launches with the step index read from the device state
 * (k = -1 for sf_gmres_givens; `scalars` = gs + the scalar block offset,
 * sf_gmres_state_doubles(R, I) - I - 8, for the MGS), so one captured CUDA
 * graph serves every Arnoldi step of a solve; both are no-ops once the
 * cycle is done. */
int sf_gmres_mgs_dk(double *V, int64_t ld, const double *scalars, double *w, int64_t n,
                    double *hcol, int R, double *work, void *stream);
int sf_gmres_update(const double *V, int64_t ld, double *gs, int R, double *x, int64_t n,
                    void *stream);

/* Near-field map construction on the device.
 * sf_near_search: (fiber, target) pairs whose minimum node distance is below
 * the fiber's shell 1.5 L/p, target outside the fiber's group
 * (system.py:564-577); pairs (cap,2) as [l, t], *count = number found (may
 * exceed cap: call again with a larger buffer); order unspecified.
 * center/bound/shell (nf): node centroid, max node distance + shell, shell.
 * sf_near_fiber_weights: W (npairs,3,3n) = near_fiber_weights -
 * plain_fiber_weights (fiber.py:514-575) for pairs (pt[e], pl[e]); Cmat (n,n)
 * maps nodal values to Chebyshev coefficients, gl = 10 Gauss-Legendre nodes
 * then weights on [-1,1]; info (npairs): 0 ok, 1 target inside the fiber
 * (InsideFiberError, fiber.py:527-528), 2 panel overflow.  n <= 128. */
int sf_near_search(const double *trg, const int64_t *tgrp, int64_t nt, const double *X,
                   int64_t nf, int64_t n, const double *center, const double *bound,
                   const double *shell, int64_t cap, int64_t *pairs,
                   unsigned long long *count, void *stream);
int sf_near_fiber_weights(const int64_t *pt, const int64_t *pl, int64_t npairs,
                          const double *targets, const double *X, const double *s_alpha,
                          const double *wcc, const double *Cmat, const double *nodes,
                          const double *gl, const double *eps, const double *L, int64_t n,
                          double mu, int include_doublet, double *W, int *info, void *stream);

/* Near-surface correction maps Wnear - Wplain (body.py:479-519,
 * system.py:588-613) for npairs (target, surface) pairs of ONE surface.
 * Coarse mesh: nt x nph patches of 16 Gauss-Legendre nodes (patch-major);
 * fine mesh: the same surface at (f nt) x (f nph) patches; fcoef (Nf,8) the
 * Lagrange coefficients (theta then phi) of each fine node in its coarse
 * patch.  Per pair (host-computed, body.py:371-423 and :479-519): target,
 * nearest surface point x0, the three off-surface points pts (3,3), their
 * Lagrange weights ell (4), jump (1/mu inside a periphery, else 0), the
 * fine patch index and 16 coefficients of the interpolation row at x0.
 * f = 1 with the coarse mesh as "fine" mesh gives the on-surface map.
 * work >= npairs * (9 + 148*9) doubles; W (npairs, 3, 3 Nc). */
int sf_near_surface_weights(const double *cnodes, const double *cnrm, const double *cw,
                            int64_t nt, int64_t nph, const double *fnodes, const double *fnrm,
                            const double *fw, const double *fcoef, int f, int64_t npairs,
                            const double *trg, const double *x0, const double *pts,
                            const double *ell, const double *jump, const int64_t *r0patch,
                            const double *r0coef, double mu, double *work, double *W,
                            void *stream);

/* Near-field correction apply (system.py:702-707): for every entry e,
 * u[t_e] += W_e (3 x 3 m_e) . x[off_e : off_e + 3 m_e].  Entries must be
 * grouped by target (row_ptr CSR over `nrows` distinct targets rows[]);
 * within a target they are applied in list order.  W is packed per entry at
 * w_off[e] (doubles). */
int sf_near_apply(const int64_t *row_ptr, const int64_t *rows, int64_t nrows,
                  const int64_t *w_off, const int64_t *x_off, const int64_t *x_len,
                  const double *W, const double *x, double *u, void *stream);

/* ---------------------------------------------------------------------------
 * Host-buffer drop-ins (copy in, compute, copy out, synchronise).
 * ------------------------------------------------------------------------- */
int sf_host_stokeslet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                          const double *src, const int64_t *sgrp, int64_t ns,
                          const double *f, double pref, double *out, int64_t *bad);
int sf_host_doublet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                        const double *src, const int64_t *sgrp, int64_t ns,
                        const double *f, double pref, double *out, int64_t *bad);
int sf_host_sbt_pair(const double *trg, const int64_t *tgrp, int64_t nt,
                     const double *src, const int64_t *sgrp, int64_t ns,
                     const double *f, const double *dcoef, double pref, int mode,
                     double *out, int64_t *bad);
int sf_host_stresslet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                          const double *src, const int64_t *sgrp, int64_t ns,
                          const double *nrm, const double *qw, double pref,
                          double *out, int64_t *bad);
int sf_host_stresslet_sum_subtracted(const double *nodes, const double *nrm,
                                     const double *w, const double *q, int64_t n,
                                     double pref, double *out);
int sf_host_stresslet_rowsum(const double *nodes, const double *nrm,
                             const double *w, int64_t n, double pref, double *out);
int sf_host_kdelta_matrix(const double *X, const double *s, const double *s_alpha,
                          const double *tang, const double *w, int64_t n,
                          double delta, double pref, double *K);

/* ---------------------------------------------------------------------------
 * Octree Stokeslet summation: the reference's TreeSummation backend
 * (system.py:108-224).  Sources/strengths src, f (ns,3) permuted so node k
 * owns [nbeg[k], nend[k]); children of k are nodes first_child[k] ..
 * first_child[k] + nchild[k] - 1 in octant order (host-built topology,
 * system.py:112-140).  Moments, traversal with the reference's opening test
 * (theta, cell_tolerance, C2 = 16) and the same-group subtraction run on the
 * device; group g's sources are gsrc/gf[gbeg[g] .. gend[g]).  work >=
 * sf_tree_work_doubles(nnodes) doubles; out (nt,3) overwritten.
 * ------------------------------------------------------------------------- */
int sf_tree_stokeslet(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                      const double *f, int64_t ns, const int64_t *nbeg, const int64_t *nend,
                      const int64_t *first_child, const int *nchild, int64_t nnodes,
                      const double *gsrc, const double *gf, const int64_t *gbeg,
                      const int64_t *gend, int64_t ngroups, double theta, double cell_tolerance,
                      double mu, double *work, double *out, void *stream);
int64_t sf_tree_work_doubles(int64_t nnodes);

/* ---------------------------------------------------------------------------
 * Measurement helpers.
 * ------------------------------------------------------------------------- */

/* FP64 DFMA throughput microbenchmark: runs `iters` dependent-chain DFMA
 * iterations on every resident thread; writes achieved DFMA FLOP/s (2 per
 * DFMA) into *flops.  Used as the roofline denominator. */
int sf_dfma_peak(int64_t iters, double *flops, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* SF_B200_H */
