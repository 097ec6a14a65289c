// sf_internal.h — library-internal declarations shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <functional>
#include <stddef.h>
#include <stdint.h>

#include "../../include/sf_b200.h"

namespace sf {

// Records a CUDA error (if any) from the last launch; returns SF_OK/SF_ECUDA.
int check_launch(const char *what);
int set_error(int code, const char *fmt, ...);

// Grow-only, stream-ordered device scratch.  One instance per stream; slots
// are independent buffers.  Steady-state calls allocate nothing.
class Workspace {
   public:
    // slots: 0-2 pair engine, 3-5 symmetric kernels, 6 skipped-pair scratch,
    // 7-10 cross kernel, 11 side-stream stresslet sum, 12 symmetric waves
    static constexpr int kSlots = 14;
    void *get(int slot, size_t bytes, cudaStream_t st);
    void release();   // frees every slot (the caller synchronised the device)
    size_t bytes() const {
        size_t b = 0;
        for (int k = 0; k < kSlots; ++k) b += cap_[k];
        return b;
    }
    ~Workspace();

   private:
    void *ptr_[kSlots] = {};
    size_t cap_[kSlots] = {};
};
Workspace &workspace_for(cudaStream_t st);
size_t workspace_bytes_total();
void workspace_release_all();   // synchronises each device, frees every workspace slot

// Side streams of one caller stream (keyed by device and stream), forked from
// and joined back into it with events; created once per process.  done[0]
// belongs to the caller stream, done[k + 1] to s[k].  Used under stream
// capture too: every side stream first waits on `fork`, recorded on the
// capturing stream, and the caller stream waits on the side work it needs.
struct SidePool {
    static constexpr int kStreams = 3;
    cudaStream_t s[kStreams] = {};
    cudaEvent_t fork = nullptr;
    cudaEvent_t done[kStreams + 1] = {};
};
SidePool *side_pool_for(cudaStream_t st);

int pairs_sbt(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
              const int64_t *sgrp, int64_t ns, const double *f, const double *dcoef, double pref,
              int mode, double *out, int64_t *bad, cudaStream_t st, Workspace &ws);
int pairs_doublet_only(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                       const int64_t *sgrp, int64_t ns, const double *f, double pref, double *out,
                       int64_t *bad, cudaStream_t st, Workspace &ws);
int pairs_stresslet(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                    const int64_t *sgrp, int64_t ns, const double *nrm, const double *qw,
                    double pref, double *out, int64_t *bad, cudaStream_t st, Workspace &ws,
                    const double *wsrc = nullptr, int accumulate = 0);
int pairs_dl_subtracted(const double *nodes, const double *nrm, const double *w, const double *q,
                        int64_t n, double pref, double *out, cudaStream_t st, Workspace &ws);
int pairs_rowsum(const double *nodes, const double *nrm, const double *w, int64_t n, double pref,
                 double *out, cudaStream_t st, Workspace &ws);

int fiber_kdelta_build(const double *X, const double *s, const double *s_alpha,
                       const double *tang, const double *w, int64_t nf, int64_t n,
                       const double *delta, double pref, double *K, cudaStream_t st);
int fiber_self_apply(const double *K, const double *tang, const double *c_log, double c_two,
                     const double *f, int64_t nf, int64_t n, int accumulate, double *u,
                     cudaStream_t st);
int fiber_geometry(const double *X, int64_t nf, int64_t n, const double *D, const double *S,
                   const double *wcc, double delta_ratio, double *s, double *s_alpha,
                   double *tang, double *wnode, double *L, double *delta, int *degenerate,
                   cudaStream_t st);
int pairs_sbt_weighted(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                       const int64_t *sgrp, int64_t ns, const double *f, const double *wsrc,
                       const double *dcoef, double pref, int mode, double *out, int64_t *bad,
                       cudaStream_t st, Workspace &ws, int accumulate = 0);
int pair_split(int64_t nt, int64_t ns);
int pairs_sbt_symmetric(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                        const double *f, const double *w, const double *dcoef, double pref,
                        double *out, int64_t *bad, int accumulate, cudaStream_t st,
                        Workspace &ws, int mode = SF_MODE_FP64,
                        const std::function<int()> *after_pack = nullptr);
bool use_symmetric(int mode, int64_t N);
int pairs_sbt_symmetric_shard(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                              const double *f, const double *w, const double *dcoef, double pref,
                              int rank, int world, double *out, int64_t *bad, int accumulate,
                              cudaStream_t st, Workspace &ws, int mode = SF_MODE_FP64,
                              const std::function<int()> *after_pack = nullptr);
int pairs_sbt_symmetric_tasks(const double *x, const int64_t *grp, int64_t N, int64_t group_size,
                              const double *f, const double *w, const double *dcoef, double pref,
                              int64_t t0, int64_t ntasks, double *out, int64_t *bad,
                              int accumulate, cudaStream_t st, Workspace &ws, int mode,
                              const std::function<int()> *after_pack = nullptr);
int64_t sym_task_total(int64_t N, int64_t group_size, int mode);
int64_t sym_launch_count_range(int64_t N, int64_t group_size, int mode, int64_t t0,
                               int64_t ntasks);
int sym_task_costs(const double *x, const int64_t *grp, int64_t N, int64_t group_size, int mode,
                   double c_checked, double c_diag, double *cost, cudaStream_t st, Workspace &ws);
int add_counter(int64_t *dst, const int64_t *src, cudaStream_t st);
int sym_unit_size(int64_t N, int64_t group_size, int mode);
int64_t sym_launch_count(int64_t N, int64_t group_size, int mode, int rank, int world);
void sym_set_waves(int64_t bytes, int streams);
// fiber points (A) x surface nodes (B), both directions per pair (sf_cross.cu)
int pairs_cross(const double *xa, const double *fa, const double *wa, const double *dcoef,
                int64_t NA, const double *xb, const double *qb, const double *wb,
                const double *nb, int64_t NB, double pref_a, double pref_b, double *out_a,
                int accumulate_a, double *out_b, int accumulate_b, int64_t *bad_a,
                int64_t *bad_b, cudaStream_t st, Workspace &ws);
bool use_cross(int64_t NA, int64_t NB);
// symmetric on-surface subtracted double layer for large meshes (sf_dlsym.cu)
bool use_dl_symmetric(int64_t n);
int pairs_dl_subtracted_symmetric(const double *nodes, const double *nrm, const double *w,
                                  const double *q, int64_t n, double pref, double *out,
                                  cudaStream_t st, Workspace &ws, int rank = 0, int world = 1);
int64_t sym_task_range(int64_t G, int64_t N, int64_t M, int rank, int world, int64_t *count);
int near_apply(const int64_t *row_ptr, const int64_t *rows, int64_t nrows, const int64_t *w_off,
               const int64_t *x_off, const int64_t *x_len, const double *W, const double *x,
               double *u, cudaStream_t st);

}  // namespace sf
