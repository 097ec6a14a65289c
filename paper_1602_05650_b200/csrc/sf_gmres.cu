// sf_gmres.cu — the Hessenberg / Givens bookkeeping of restarted GMRES
// (solver.py:444-516 of the reference) on the device, sm_100a.
//
// The Krylov basis, the Arnoldi vector and the Gram-Schmidt coefficients
// already live on the device (sf_gmres_mgs writes h_{0..k+1} and |w| into
// hcol).  This file keeps the rest of one Arnoldi step there too -- the
// rotations of the new Hessenberg column, the new rotation, the residual
// estimate g, the convergence and breakdown tests, the per-iteration residual
// history -- and the restart update x += V_k^T H_k^-1 g_k.  The host reads one
// small status record per iteration (copied asynchronously into pinned
// memory, consumed with a lag) instead of the whole column, so it can queue
// the next matvec before the current one has finished.
//
// A step whose status is already "done" (converged, broke down, cycle full
// or iteration cap reached) is a no-op: an Arnoldi step queued speculatively
// behind the converged one changes nothing the solution reads (it would only
// touch column k+1 of H, g[k+1..k+2] and V[k+2]).
//
// State layout (doubles), R = restart, I = iteration cap:
//   H[(R+1) x R] row-major | cs[R] | sn[R] | g[R+1] | y[R] | scalars[8] | hist[I]
// scalars: k (columns of this cycle), iters (total), done, rel, beta0, tol,
//          max_iterations, breakdown.
#include <cmath>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {
namespace {

enum { S_K = 0, S_ITERS, S_DONE, S_REL, S_BETA0, S_TOL, S_MAXIT, S_BREAK, S_N };

struct GState {
    double *H, *cs, *sn, *g, *y, *s, *hist;
    int R;
};

__device__ __forceinline__ GState gstate(double *gs, int R) {
    GState v;
    v.R = R;
    v.H = gs;
    v.cs = v.H + (int64_t)(R + 1) * R;
    v.sn = v.cs + R;
    v.g = v.sn + R;
    v.y = v.g + R + 1;
    v.s = v.y + R;
    v.hist = v.s + S_N;
    return v;
}

// iteration-start state of a solve: iters = 0, tolerances
__global__ void gmres_reset_kernel(double *gs, int R, double beta0, double tol, int maxit) {
    GState G = gstate(gs, R);
    G.s[S_K] = 0.0;
    G.s[S_ITERS] = 0.0;
    G.s[S_DONE] = 0.0;
    G.s[S_REL] = 0.0;
    G.s[S_BETA0] = beta0;
    G.s[S_TOL] = tol;
    G.s[S_MAXIT] = (double)maxit;
    G.s[S_BREAK] = 0.0;
}

// a new cycle (solver.py:470-480): g = beta e_0, k = 0; V_0 = r / beta
__global__ void gmres_cycle_kernel(double *gs, int R, const double *__restrict__ beta) {
    GState G = gstate(gs, R);
    const int t = threadIdx.x;
    const double b = beta[0];
    for (int j = t; j <= R; j += blockDim.x) G.g[j] = j == 0 ? b : 0.0;
    if (t == 0) {
        G.s[S_K] = 0.0;
        G.s[S_DONE] = 0.0;
        G.s[S_BREAK] = 0.0;
    }
}

// One Arnoldi step's Hessenberg bookkeeping (solver.py:484-505), one thread:
// hcol = [h_0 .. h_k, |w_orth|, ..., wnorm at R+1] from sf_gmres_mgs.
__global__ void gmres_givens_kernel(const double *__restrict__ hcol, double *gs, int R, int k,
                                    double *__restrict__ status) {
    GState G = gstate(gs, R);
    if (k < 0) k = (int)G.s[S_K];          // step index from the device (graph replays)
    if (G.s[S_DONE] == 0.0 && (int)G.s[S_K] == k && k < R) {
        const double wnorm = hcol[R + 1];
        double *H = G.H;
        for (int j = 0; j <= k + 1; ++j) H[(int64_t)j * R + k] = hcol[j];
        for (int j = 0; j < k; ++j) {
            const double a = H[(int64_t)j * R + k], b = H[(int64_t)(j + 1) * R + k];
            const double tmp = G.cs[j] * a + G.sn[j] * b;
            H[(int64_t)(j + 1) * R + k] = -G.sn[j] * a + G.cs[j] * b;
            H[(int64_t)j * R + k] = tmp;
        }
        const double hkk = H[(int64_t)k * R + k], hk1 = H[(int64_t)(k + 1) * R + k];
        const double denom = hypot(hkk, hk1);
        G.cs[k] = denom != 0.0 ? hkk / denom : 1.0;
        G.sn[k] = denom != 0.0 ? hk1 / denom : 0.0;
        H[(int64_t)k * R + k] = denom;
        G.g[k + 1] = -G.sn[k] * G.g[k];
        G.g[k] = G.cs[k] * G.g[k];
        const int iters = (int)G.s[S_ITERS] + 1;
        const double rel = fabs(G.g[k + 1]) / G.s[S_BETA0];
        G.hist[iters - 1] = rel;
        const bool breakdown = hk1 <= 1e-12 * fmax(wnorm, 1e-300);
        G.s[S_ITERS] = (double)iters;
        G.s[S_REL] = rel;
        G.s[S_K] = (double)(k + 1);
        G.s[S_BREAK] = breakdown ? 1.0 : 0.0;
        if (rel <= G.s[S_TOL] || breakdown || k + 1 >= R || iters >= (int)G.s[S_MAXIT])
            G.s[S_DONE] = 1.0;
    }
    if (status) {
        status[0] = G.s[S_DONE];
        status[1] = G.s[S_ITERS];
        status[2] = G.s[S_REL];
        status[3] = G.s[S_K];
    }
}

// y = triu(H[:k,:k])^-1 g[:k] by back substitution (solver.py:507), one thread
__global__ void gmres_trisolve_kernel(double *gs, int R) {
    GState G = gstate(gs, R);
    const int k = (int)G.s[S_K];
    for (int i = k - 1; i >= 0; --i) {
        double s = G.g[i];
        for (int j = i + 1; j < k; ++j) s -= G.H[(int64_t)i * R + j] * G.y[j];
        G.y[i] = s / G.H[(int64_t)i * R + i];
    }
}

// x += sum_{j < k} y_j V_j, k and y read from the state (fixed j order)
__global__ void gmres_combine_kernel(const double *__restrict__ V, int64_t ld,
                                     const double *__restrict__ gs_c, int R,
                                     double *__restrict__ x, int64_t n) {
    GState G = gstate(const_cast<double *>(gs_c), R);
    const int k = (int)G.s[S_K];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s = fma(G.y[j], V[(int64_t)j * ld + i], s);
        x[i] += s;
    }
}

// V_0 = r / beta (beta a device scalar)
__global__ void gmres_scale_kernel(const double *__restrict__ r, const double *__restrict__ beta,
                                   double *__restrict__ v, int64_t n) {
    const double inv = 1.0 / beta[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = r[i] * inv;
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 8192 ? 8192 : g));
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" {

int64_t sf_gmres_state_doubles(int R, int max_iterations) {
    if (R < 1 || max_iterations < 1) return 0;
    return (int64_t)(R + 1) * R + 2 * R + (R + 1) + R + S_N + max_iterations;
}

int sf_gmres_reset(double *gs, int R, int max_iterations, double beta0, double tol,
                   void *stream) {
    if (!gs || R < 1 || max_iterations < 1) return set_error(SF_EINVAL, "bad GMRES state");
    gmres_reset_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(gs, R, beta0, tol, max_iterations);
    return check_launch("gmres_reset_kernel");
}

int sf_gmres_cycle(double *gs, int R, const double *beta, const double *r, double *V0, int64_t n,
                   void *stream) {
    if (!gs || !beta || R < 1 || n < 0) return set_error(SF_EINVAL, "bad GMRES cycle");
    cudaStream_t st = (cudaStream_t)stream;
    gmres_cycle_kernel<<<1, 64, 0, st>>>(gs, R, beta);
    int rc = check_launch("gmres_cycle_kernel");
    if (rc || n == 0) return rc;
    gmres_scale_kernel<<<grid_for(n), 256, 0, st>>>(r, beta, V0, n);
    return check_launch("gmres_scale_kernel");
}

int sf_gmres_givens(const double *hcol, double *gs, int R, int k, double *status, void *stream) {
    if (!hcol || !gs || k < -1 || k >= R) return set_error(SF_EINVAL, "bad Givens step");
    gmres_givens_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(hcol, gs, R, k, status);
    return check_launch("gmres_givens_kernel");
}

int sf_gmres_update(const double *V, int64_t ld, double *gs, int R, double *x, int64_t n,
                    void *stream) {
    if (!gs || R < 1 || n < 0) return set_error(SF_EINVAL, "bad GMRES update");
    cudaStream_t st = (cudaStream_t)stream;
    gmres_trisolve_kernel<<<1, 1, 0, st>>>(gs, R);
    int rc = check_launch("gmres_trisolve_kernel");
    if (rc || n == 0) return rc;
    gmres_combine_kernel<<<grid_for(n), 256, 0, st>>>(V, ld, gs, R, x, n);
    return check_launch("gmres_combine_kernel");
}

}  // extern "C"
