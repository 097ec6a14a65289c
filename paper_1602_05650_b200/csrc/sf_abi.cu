// sf_abi.cu — the extern "C" boundary (include/sf_b200.h): argument checks,
// error reporting, per-stream workspaces, host-buffer drop-ins, and the FP64
// DFMA peak microbenchmark used as the roofline denominator.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "sf_common.cuh"
#include "sf_internal.h"

namespace sf {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return SF_OK;
}

void *Workspace::get(int slot, size_t bytes, cudaStream_t st) {
    if (slot < 0 || slot >= kSlots) return nullptr;
    if (bytes == 0) bytes = 16;
    if (cap_[slot] >= bytes) return ptr_[slot];
    // growing inside a stream capture would cache a graph-owned pointer:
    // callers warm the path up (one uncaptured call) before capturing it
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        set_error(SF_ENOMEM, "workspace slot %d must grow to %zu bytes during stream capture; "
                  "run the call once before capturing it", slot, bytes);
        return nullptr;
    }
    if (ptr_[slot]) cudaFreeAsync(ptr_[slot], st);
    size_t cap = bytes + bytes / 4;
    void *p = nullptr;
    if (cudaMallocAsync(&p, cap, st) != cudaSuccess) {
        cudaGetLastError();
        ptr_[slot] = nullptr;
        cap_[slot] = 0;
        set_error(SF_ENOMEM, "workspace allocation of %zu bytes failed", cap);
        return nullptr;
    }
    ptr_[slot] = p;
    cap_[slot] = cap;
    return p;
}

Workspace::~Workspace() {}

void Workspace::release() {
    for (int k = 0; k < kSlots; ++k) {
        if (ptr_[k]) cudaFree(ptr_[k]);
        ptr_[k] = nullptr;
        cap_[k] = 0;
    }
}

// Per-stream state is keyed by (device, stream): the legacy default stream
// handle 0 (and per-thread default streams) is the same value on every
// device, so a stream handle alone does not identify one device's queue.
static uint64_t stream_key(cudaStream_t st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    return ((uint64_t)(uintptr_t)st << 8) ^ (uint64_t)(unsigned)dev;
}

static std::mutex g_ws_mu;
static std::unordered_map<uint64_t, Workspace *> *g_ws = nullptr;

Workspace &workspace_for(cudaStream_t st) {
    const uint64_t key = stream_key(st);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (!g_ws) g_ws = new std::unordered_map<uint64_t, Workspace *>();
    auto it = g_ws->find(key);
    if (it != g_ws->end()) return *it->second;
    Workspace *w = new Workspace();
    (*g_ws)[key] = w;
    return *w;
}

size_t workspace_bytes_total() {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    size_t b = 0;
    if (g_ws)
        for (auto &kv : *g_ws) b += kv.second->bytes();
    return b;
}

void workspace_release_all() {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (!g_ws) return;
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : *g_ws) {
        const int dev = (int)(kv.first & 0xff);
        if (cudaSetDevice(dev) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess)
            kv.second->release();
        cudaGetLastError();
    }
    cudaSetDevice(cur);
}

static std::mutex g_side_mu;
static std::unordered_map<uint64_t, SidePool *> *g_side = nullptr;

SidePool *side_pool_for(cudaStream_t st) {
    const uint64_t key = stream_key(st);
    std::lock_guard<std::mutex> lk(g_side_mu);
    if (!g_side) g_side = new std::unordered_map<uint64_t, SidePool *>();
    auto it = g_side->find(key);
    if (it != g_side->end()) return it->second;
    SidePool *p = new SidePool();
    bool ok = cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&p->done[0], cudaEventDisableTiming) == cudaSuccess;
    // SF_SIDE_FIRST=1 (A/B, see sf_operator.cu) also puts the last stream,
    // which carries the operator's overlapping sums, at the highest priority
    static const bool prio = [] {
        const char *e = getenv("SF_SIDE_FIRST");
        return e && atoi(e) == 1;
    }();
    int least = 0, greatest = 0;
    if (prio && cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
        cudaGetLastError();
        greatest = 0;
    }
    for (int k = 0; ok && k < SidePool::kStreams; ++k) {
        const int pr = (prio && k == SidePool::kStreams - 1) ? greatest : 0;
        ok = cudaStreamCreateWithPriority(&p->s[k], cudaStreamNonBlocking, pr) == cudaSuccess &&
             cudaEventCreateWithFlags(&p->done[k + 1], cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        delete p;
        return nullptr;  // no side streams: callers run in order on st
    }
    (*g_side)[key] = p;
    return p;
}

// ---- host-buffer staging (drop-in path): grow-only device + pinned buffers
struct HostStage {
    cudaStream_t st = nullptr;
    void *dev[12] = {};
    size_t cap[12] = {};
    std::mutex mu;
    int init() {
        if (st) return SF_OK;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            return set_error(SF_ECUDA, "stream create failed: %s",
                             cudaGetErrorString(cudaGetLastError()));
        return SF_OK;
    }
    void *buf(int i, size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (cap[i] >= bytes) return dev[i];
        if (dev[i]) cudaFree(dev[i]);
        dev[i] = nullptr;
        cap[i] = 0;
        if (cudaMalloc(&dev[i], bytes) != cudaSuccess) {
            cudaGetLastError();
            set_error(SF_ENOMEM, "device staging allocation of %zu bytes failed", bytes);
            return nullptr;
        }
        cap[i] = bytes;
        return dev[i];
    }
};
static HostStage g_stage;

}  // namespace sf

using namespace sf;

#define SF_REQUIRE(cond, msg) \
    do {                      \
        if (!(cond)) return set_error(SF_EINVAL, "%s", msg); \
    } while (0)

extern "C" {

int sf_abi_version(void) { return 1; }
const char *sf_last_error(void) { return g_err; }

int sf_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

int sf_stokeslet_sum(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                     const int64_t *sgrp, int64_t ns, const double *f, double pref, double *out,
                     int64_t *bad, void *stream) {
    SF_REQUIRE(nt >= 0 && ns >= 0, "negative size");
    SF_REQUIRE(nt == 0 || (trg && out), "null target/output pointer");
    SF_REQUIRE(ns == 0 || (src && f), "null source pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_sbt(trg, tgrp, nt, src, sgrp, ns, f, nullptr, pref, SF_MODE_FP64, out, bad, st,
                     workspace_for(st));
}

int sf_sbt_pair(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                const int64_t *sgrp, int64_t ns, const double *f, const double *dcoef,
                double pref, int mode, double *out, int64_t *bad, void *stream) {
    SF_REQUIRE(nt >= 0 && ns >= 0, "negative size");
    SF_REQUIRE(nt == 0 || (trg && out), "null target/output pointer");
    SF_REQUIRE(ns == 0 || (src && f), "null source pointer");
    SF_REQUIRE(mode == SF_MODE_FP64 || mode == SF_MODE_FP32C, "unknown mode");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_sbt(trg, tgrp, nt, src, sgrp, ns, f, dcoef, pref, mode, out, bad, st,
                     workspace_for(st));
}

int sf_stresslet_sum(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                     const int64_t *sgrp, int64_t ns, const double *nrm, const double *qw,
                     double pref, double *out, int64_t *bad, void *stream) {
    SF_REQUIRE(nt >= 0 && ns >= 0, "negative size");
    SF_REQUIRE(nt == 0 || (trg && out), "null target/output pointer");
    SF_REQUIRE(ns == 0 || (src && nrm && qw), "null source pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_stresslet(trg, tgrp, nt, src, sgrp, ns, nrm, qw, pref, out, bad, st,
                           workspace_for(st));
}

int sf_stresslet_sum_subtracted(const double *nodes, const double *nrm, const double *w,
                                const double *q, int64_t n, double pref, double *out,
                                void *stream) {
    SF_REQUIRE(n >= 0, "negative size");
    SF_REQUIRE(n == 0 || (nodes && nrm && w && q && out), "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_dl_subtracted(nodes, nrm, w, q, n, pref, out, st, workspace_for(st));
}

int sf_stresslet_sum_subtracted_partial(const double *nodes, const double *nrm, const double *w,
                                        const double *q, int64_t n, double pref, int rank,
                                        int world, double *out, void *stream) {
    SF_REQUIRE(n >= 0 && world >= 1 && rank >= 0 && rank < world, "bad sizes");
    SF_REQUIRE(n == 0 || (nodes && nrm && w && q && out), "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_dl_subtracted_symmetric(nodes, nrm, w, q, n, pref, out, st, workspace_for(st),
                                         rank, world);
}

int sf_stresslet_rowsum(const double *nodes, const double *nrm, const double *w, int64_t n,
                        double pref, double *out, void *stream) {
    SF_REQUIRE(n >= 0, "negative size");
    SF_REQUIRE(n == 0 || (nodes && nrm && w && out), "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_rowsum(nodes, nrm, w, n, pref, out, st, workspace_for(st));
}

int sf_kdelta_build_batched(const double *X, const double *s, const double *s_alpha,
                            const double *tang, const double *w, int64_t nf, int64_t n,
                            const double *delta, double pref, double *K, void *stream) {
    SF_REQUIRE(nf >= 0 && n >= 2, "bad fiber sizes");
    SF_REQUIRE(nf == 0 || (X && s && s_alpha && tang && w && delta && K), "null pointer");
    return fiber_kdelta_build(X, s, s_alpha, tang, w, nf, n, delta, pref, K,
                              (cudaStream_t)stream);
}

int sf_self_apply_batched(const double *K, const double *tang, const double *c_log,
                          double c_two, const double *f, int64_t nf, int64_t n, int accumulate,
                          double *u, void *stream) {
    SF_REQUIRE(nf >= 0 && n >= 2, "bad fiber sizes");
    SF_REQUIRE(nf == 0 || (tang && c_log && f && u), "null pointer");
    return fiber_self_apply(K, tang, c_log, c_two, f, nf, n, accumulate, u,
                            (cudaStream_t)stream);
}

int sf_near_apply(const int64_t *row_ptr, const int64_t *rows, int64_t nrows,
                  const int64_t *w_off, const int64_t *x_off, const int64_t *x_len,
                  const double *W, const double *x, double *u, void *stream) {
    SF_REQUIRE(nrows >= 0, "negative size");
    SF_REQUIRE(nrows == 0 || (row_ptr && rows && w_off && x_off && x_len && W && x && u),
               "null pointer");
    return near_apply(row_ptr, rows, nrows, w_off, x_off, x_len, W, x, u, (cudaStream_t)stream);
}

}  // extern "C"

extern "C" int sf_doublet_sum(const double *trg, const int64_t *tgrp, int64_t nt,
                              const double *src, const int64_t *sgrp, int64_t ns,
                              const double *f, double pref, double *out, int64_t *bad,
                              void *stream) {
    SF_REQUIRE(nt >= 0 && ns >= 0, "negative size");
    SF_REQUIRE(nt == 0 || (trg && out), "null target/output pointer");
    SF_REQUIRE(ns == 0 || (src && f), "null source pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_doublet_only(trg, tgrp, nt, src, sgrp, ns, f, pref, out, bad, st,
                              workspace_for(st));
}

extern "C" int sf_fiber_geometry_batched(const double *X, int64_t nf, int64_t n,
                                         const double *D, const double *S, const double *wcc,
                                         double delta_ratio, double *s, double *s_alpha,
                                         double *tang, double *wnode, double *L, double *delta,
                                         int *degenerate, void *stream) {
    SF_REQUIRE(nf >= 0 && n >= 2, "bad fiber sizes");
    SF_REQUIRE(nf == 0 || (X && D && S && wcc && s && s_alpha && tang && wnode && L),
               "null pointer");
    SF_REQUIRE(delta_ratio <= 0 || delta, "delta output required when delta_ratio > 0");
    return fiber_geometry(X, nf, n, D, S, wcc, delta_ratio, s, s_alpha, tang, wnode, L, delta,
                          degenerate, (cudaStream_t)stream);
}

extern "C" int sf_fiber_hi_apply(const double *X, const int64_t *grp, int64_t nf, int64_t n,
                                 int64_t t_fiber0, int64_t t_nfibers, const double *wnode,
                                 const double *dcoef, double pref, int mode, const double *K,
                                 const double *tang, const double *c_log, double c_two,
                                 const int64_t *near_row_ptr, const int64_t *near_rows,
                                 int64_t near_nrows, const int64_t *near_w_off,
                                 const int64_t *near_x_off, const int64_t *near_x_len,
                                 const double *near_W, const double *f, double *out_nl,
                                 double *out_self, int64_t *bad, void *stream) {
    SF_REQUIRE(nf >= 0 && n >= 2 && near_nrows >= 0, "bad sizes");
    SF_REQUIRE(t_fiber0 >= 0 && t_nfibers >= 0 && t_fiber0 + t_nfibers <= nf,
               "target fiber range outside [0, nf)");
    SF_REQUIRE(nf == 0 || (X && wnode && f && out_nl), "null pointer");
    SF_REQUIRE(!out_self || (K && tang && c_log), "self terms need K, tangents and c_log");
    SF_REQUIRE(mode == SF_MODE_FP64 || mode == SF_MODE_FP32C || mode == SF_MODE_FP64_DIRECT,
               "unknown mode");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = nf * n;
    const int64_t t0 = t_fiber0 * n, nt = t_nfibers * n;
    int rc;
    if (t_fiber0 == 0 && t_nfibers == nf && use_symmetric(mode, N))
        rc = pairs_sbt_symmetric(X, grp, N, n, f, wnode, dcoef, pref, out_nl, bad, 0, st,
                                 workspace_for(st), mode);
    else
        rc = pairs_sbt_weighted(X + 3 * t0, grp ? grp + t0 : nullptr, nt, X, grp, N, f, wnode,
                                dcoef, pref, mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64,
                                out_nl, bad, st, workspace_for(st));
    if (rc) return rc;
    if (near_nrows > 0) {
        rc = near_apply(near_row_ptr, near_rows, near_nrows, near_w_off, near_x_off, near_x_len,
                        near_W, f, out_nl, st);
        if (rc) return rc;
    }
    if (out_self)
        rc = fiber_self_apply(K, tang + 3 * t0, c_log + t_fiber0, c_two, f + 3 * t0, t_nfibers,
                              n, 0, out_self, st);
    return rc;
}

extern "C" int sf_pair_split(int64_t nt, int64_t ns) { return sf::pair_split(nt, ns); }

extern "C" int64_t sf_workspace_bytes(void) { return (int64_t)sf::workspace_bytes_total(); }

extern "C" int sf_workspace_release(void) {
    sf::workspace_release_all();
    return SF_OK;
}

extern "C" int sf_sym_set_waves(int64_t bytes, int streams) {
    sf::sym_set_waves(bytes, streams);
    return SF_OK;
}

extern "C" int64_t sf_sym_launch_count(int64_t N, int64_t group_size, int mode, int rank,
                                       int world) {
    if (N <= 0 || world < 1 || rank < 0 || rank >= world) return 0;
    return sf::sym_launch_count(N, group_size, mode, rank, world);
}

static int64_t sym_range_pairs(int64_t N, int64_t group_size, int64_t M, int64_t t0,
                               int64_t count);

extern "C" int64_t sf_sym_shard_pairs(int64_t N, int64_t group_size, int rank, int world) {
    if (N <= 0 || world < 1 || rank < 0 || rank >= world) return 0;
    const int64_t M = sf::sym_unit_size(N, group_size, SF_MODE_FP64);   // the FP64 task split
    const int64_t G = (N + M - 1) / M;
    int64_t count = 0;
    const int64_t t0 = sf::sym_task_range(G, N, M, rank, world, &count);
    return sym_range_pairs(N, group_size, M, t0, count);
}

extern "C" int64_t sf_sym_range_pairs(int64_t N, int64_t group_size, int mode, int64_t t0,
                                      int64_t count) {
    if (N <= 0 || t0 < 0 || count <= 0) return 0;
    return sym_range_pairs(N, group_size, sf::sym_unit_size(N, group_size, mode), t0, count);
}

extern "C" int64_t sf_sym_unit_size(int64_t N, int64_t group_size, int mode) {
    if (N <= 0) return 0;
    return sf::sym_unit_size(N, group_size, mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64);
}

extern "C" int64_t sf_sym_task_count(int64_t N, int64_t group_size, int mode) {
    return sf::sym_task_total(N, group_size, mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64);
}

extern "C" int64_t sf_sym_range_launch_count(int64_t N, int64_t group_size, int mode, int64_t t0,
                                             int64_t count) {
    if (N <= 0 || t0 < 0 || count < 0) return 0;
    return sf::sym_launch_count_range(N, group_size,
                                      mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64, t0,
                                      count);
}

extern "C" int sf_sym_task_costs(const double *X, const int64_t *grp, int64_t N,
                                 int64_t group_size, int mode, double c_checked, double c_diag,
                                 double *cost, void *stream) {
    SF_REQUIRE(N >= 0 && (N == 0 || (X && cost)), "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    return sf::sym_task_costs(X, grp, N, group_size,
                              mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64, c_checked,
                              c_diag, cost, st, workspace_for(st));
}

extern "C" int sf_sbt_symmetric_tasks(const double *X, const int64_t *grp, int64_t N,
                                      int64_t group_size, const double *f, const double *w,
                                      const double *dcoef, double pref, int mode, int64_t t0,
                                      int64_t ntasks, double *out, int64_t *bad, void *stream) {
    SF_REQUIRE(N >= 0 && t0 >= 0 && ntasks >= 0, "bad sizes");
    SF_REQUIRE(N == 0 || (X && f && out), "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return sf::pairs_sbt_symmetric_tasks(X, grp, N, group_size, f, w, dcoef, pref, t0, ntasks, out,
                                         bad, 0, st, workspace_for(st),
                                         mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64);
}

static int64_t sym_range_pairs(int64_t N, int64_t group_size, int64_t M, int64_t t0,
                               int64_t count) {
    const int64_t G = (N + M - 1) / M;
    auto units = [&](int64_t t, int64_t &g, int64_t &h) {   // row-major {g <= h}
        int64_t r = 0, start = 0;
        while (start + (G - r) <= t) { start += G - r; ++r; }
        g = r;
        h = r + (t - start);
    };
    // ordered pairs of a task minus the same-group ones (groups are the
    // contiguous ranges [k*group_size, (k+1)*group_size))
    auto excluded = [&](int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
        if (group_size <= 0) return (int64_t)0;
        int64_t e = 0;
        for (int64_t k = a0 / group_size; k * group_size < a1; ++k) {
            const int64_t lo = k * group_size, hi = lo + group_size;
            const int64_t oa = std::min(a1, hi) - std::max(a0, lo);
            const int64_t ob = std::min(b1, hi) - std::max(b0, lo);
            if (oa > 0 && ob > 0) e += oa * ob;
        }
        return e;
    };
    int64_t g, h, pairs = 0;
    for (int64_t t = t0; t < t0 + count; ++t) {
        units(t, g, h);
        const int64_t a0 = g * M, a1 = std::min(N, a0 + M), b0 = h * M, b1 = std::min(N, b0 + M);
        const int64_t all = (a1 - a0) * (b1 - b0) - excluded(a0, a1, b0, b1);
        pairs += g != h ? 2 * all : all;
    }
    return pairs;
}

extern "C" int sf_sbt_symmetric_partial(const double *X, const int64_t *grp, int64_t N,
                                        int64_t group_size, const double *f, const double *w,
                                        const double *dcoef, double pref, int mode, int rank,
                                        int world, double *out, int64_t *bad, void *stream) {
    SF_REQUIRE(N >= 0 && world >= 1 && rank >= 0 && rank < world, "bad sizes");
    SF_REQUIRE(N == 0 || (X && f && out), "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return pairs_sbt_symmetric_shard(X, grp, N, group_size, f, w, dcoef, pref, rank, world, out,
                                     bad, 0, st, workspace_for(st),
                                     mode == SF_MODE_FP32C ? SF_MODE_FP32C : SF_MODE_FP64);
}

// ------------------------------------------------------------ host entries ----
namespace {
struct StageLock {
    std::lock_guard<std::mutex> lk;
    StageLock() : lk(g_stage.mu) {}
};

int h2d(void *dst, const void *src, size_t bytes) {
    if (!bytes) return SF_OK;
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_stage.st) != cudaSuccess)
        return check_launch("H2D copy");
    return SF_OK;
}
int d2h(void *dst, const void *src, size_t bytes) {
    if (!bytes) return SF_OK;
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_stage.st) != cudaSuccess)
        return check_launch("D2H copy");
    return SF_OK;
}
int finish() {
    if (cudaStreamSynchronize(g_stage.st) != cudaSuccess) return check_launch("synchronize");
    return SF_OK;
}
}  // namespace

#define SF_TRY(x)                 \
    do {                          \
        int rc_ = (x);            \
        if (rc_ != SF_OK) return rc_; \
    } while (0)
#define SF_BUF(var, type, idx, count)                                  \
    type *var = (type *)g_stage.buf(idx, sizeof(type) * (size_t)(count)); \
    if (!var) return SF_ENOMEM;

static int host_pairs(int kind, const double *trg, const int64_t *tgrp, int64_t nt,
                      const double *src, const int64_t *sgrp, int64_t ns, const double *a1,
                      const double *a2, double pref, int mode, double *out, int64_t *bad) {
    SF_REQUIRE(nt >= 0 && ns >= 0, "negative size");
    StageLock lock;
    SF_TRY(g_stage.init());
    SF_BUF(d_trg, double, 0, 3 * nt);
    SF_BUF(d_src, double, 1, 3 * ns);
    SF_BUF(d_a1, double, 2, 3 * ns);
    SF_BUF(d_a2, double, 3, (kind == 3 ? 3 : 1) * ns);
    SF_BUF(d_tg, int64_t, 4, nt);
    SF_BUF(d_sg, int64_t, 5, ns);
    SF_BUF(d_out, double, 6, 3 * nt);
    SF_BUF(d_bad, int64_t, 7, 1);
    SF_TRY(h2d(d_trg, trg, sizeof(double) * 3 * nt));
    SF_TRY(h2d(d_src, src, sizeof(double) * 3 * ns));
    SF_TRY(h2d(d_a1, a1, sizeof(double) * 3 * ns));
    if (a2) SF_TRY(h2d(d_a2, a2, sizeof(double) * (kind == 3 ? 3 : 1) * ns));
    if (tgrp) SF_TRY(h2d(d_tg, tgrp, sizeof(int64_t) * nt));
    if (sgrp) SF_TRY(h2d(d_sg, sgrp, sizeof(int64_t) * ns));
    const int64_t *tg = tgrp ? d_tg : nullptr;
    const int64_t *sg = sgrp ? d_sg : nullptr;
    Workspace &ws = workspace_for(g_stage.st);
    int rc;
    switch (kind) {
        case 0: rc = pairs_sbt(d_trg, tg, nt, d_src, sg, ns, d_a1, nullptr, pref, SF_MODE_FP64, d_out, d_bad, g_stage.st, ws); break;
        case 1: rc = pairs_doublet_only(d_trg, tg, nt, d_src, sg, ns, d_a1, pref, d_out, d_bad, g_stage.st, ws); break;
        case 2: rc = pairs_sbt(d_trg, tg, nt, d_src, sg, ns, d_a1, a2 ? d_a2 : nullptr, pref, mode, d_out, d_bad, g_stage.st, ws); break;
        default: rc = pairs_stresslet(d_trg, tg, nt, d_src, sg, ns, d_a1, d_a2, pref, d_out, d_bad, g_stage.st, ws); break;
    }
    SF_TRY(rc);
    SF_TRY(d2h(out, d_out, sizeof(double) * 3 * nt));
    int64_t b = 0;
    SF_TRY(d2h(&b, d_bad, sizeof(int64_t)));
    SF_TRY(finish());
    if (bad) *bad = b;
    return SF_OK;
}

extern "C" {

int sf_host_stokeslet_sum(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                          const int64_t *sgrp, int64_t ns, const double *f, double pref,
                          double *out, int64_t *bad) {
    return host_pairs(0, trg, tgrp, nt, src, sgrp, ns, f, nullptr, pref, 0, out, bad);
}
int sf_host_doublet_sum(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                        const int64_t *sgrp, int64_t ns, const double *f, double pref, double *out,
                        int64_t *bad) {
    return host_pairs(1, trg, tgrp, nt, src, sgrp, ns, f, nullptr, pref, 0, out, bad);
}
int sf_host_sbt_pair(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                     const int64_t *sgrp, int64_t ns, const double *f, const double *dcoef,
                     double pref, int mode, double *out, int64_t *bad) {
    SF_REQUIRE(mode == SF_MODE_FP64 || mode == SF_MODE_FP32C, "unknown mode");
    return host_pairs(2, trg, tgrp, nt, src, sgrp, ns, f, dcoef, pref, mode, out, bad);
}
int sf_host_stresslet_sum(const double *trg, const int64_t *tgrp, int64_t nt, const double *src,
                          const int64_t *sgrp, int64_t ns, const double *nrm, const double *qw,
                          double pref, double *out, int64_t *bad) {
    return host_pairs(3, trg, tgrp, nt, src, sgrp, ns, nrm, qw, pref, 0, out, bad);
}

int sf_host_stresslet_sum_subtracted(const double *nodes, const double *nrm, const double *w,
                                     const double *q, int64_t n, double pref, double *out) {
    SF_REQUIRE(n >= 0, "negative size");
    StageLock lock;
    SF_TRY(g_stage.init());
    SF_BUF(d_x, double, 0, 3 * n);
    SF_BUF(d_n, double, 1, 3 * n);
    SF_BUF(d_w, double, 2, n);
    SF_BUF(d_q, double, 3, 3 * n);
    SF_BUF(d_out, double, 6, 3 * n);
    SF_TRY(h2d(d_x, nodes, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_n, nrm, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_w, w, sizeof(double) * n));
    SF_TRY(h2d(d_q, q, sizeof(double) * 3 * n));
    SF_TRY(pairs_dl_subtracted(d_x, d_n, d_w, d_q, n, pref, d_out, g_stage.st,
                               workspace_for(g_stage.st)));
    SF_TRY(d2h(out, d_out, sizeof(double) * 3 * n));
    return finish();
}

int sf_host_stresslet_rowsum(const double *nodes, const double *nrm, const double *w, int64_t n,
                             double pref, double *out) {
    SF_REQUIRE(n >= 0, "negative size");
    StageLock lock;
    SF_TRY(g_stage.init());
    SF_BUF(d_x, double, 0, 3 * n);
    SF_BUF(d_n, double, 1, 3 * n);
    SF_BUF(d_w, double, 2, n);
    SF_BUF(d_out, double, 6, 9 * n);
    SF_TRY(h2d(d_x, nodes, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_n, nrm, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_w, w, sizeof(double) * n));
    SF_TRY(pairs_rowsum(d_x, d_n, d_w, n, pref, d_out, g_stage.st, workspace_for(g_stage.st)));
    SF_TRY(d2h(out, d_out, sizeof(double) * 9 * n));
    return finish();
}

int sf_host_kdelta_matrix(const double *X, const double *s, const double *s_alpha,
                          const double *tang, const double *w, int64_t n, double delta,
                          double pref, double *K) {
    SF_REQUIRE(n >= 2, "bad fiber size");
    StageLock lock;
    SF_TRY(g_stage.init());
    SF_BUF(d_X, double, 0, 3 * n);
    SF_BUF(d_s, double, 1, n);
    SF_BUF(d_sa, double, 2, n);
    SF_BUF(d_t, double, 3, 3 * n);
    SF_BUF(d_w, double, 4, n);
    SF_BUF(d_d, double, 5, 1);
    SF_BUF(d_K, double, 6, 9 * n * n);
    SF_TRY(h2d(d_X, X, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_s, s, sizeof(double) * n));
    SF_TRY(h2d(d_sa, s_alpha, sizeof(double) * n));
    SF_TRY(h2d(d_t, tang, sizeof(double) * 3 * n));
    SF_TRY(h2d(d_w, w, sizeof(double) * n));
    SF_TRY(h2d(d_d, &delta, sizeof(double)));
    SF_TRY(fiber_kdelta_build(d_X, d_s, d_sa, d_t, d_w, 1, n, d_d, pref, d_K, g_stage.st));
    SF_TRY(d2h(K, d_K, sizeof(double) * 9 * n * n));
    return finish();
}

}  // extern "C"

// ------------------------------------------------------------- DFMA peak ----
namespace sf {
// 8 independent DFMA chains per thread; 2 flops per DFMA.
__global__ void dfma_peak_kernel(int64_t iters, double seed, double *sink) {
    double a0 = seed + threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
    double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
    const double b = 0.999999999, c = 1e-10;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 12345.678) sink[0] = r;
}
}  // namespace sf

extern "C" int sf_dfma_peak(int64_t iters, double *flops, double *ms) {
    int sms = sf_device_sm_count();
    if (sms <= 0) return set_error(SF_ENODEV, "no CUDA device");
    double *sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return check_launch("malloc");
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_peak_kernel<<<blocks, threads>>>(iters / 10 + 1, 1.0, sink);  // warm-up
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(iters, 1.0, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    int rc = check_launch("dfma_peak_kernel");
    if (rc) return rc;
    const double n_dfma = (double)blocks * threads * (double)iters * 64.0;
    if (flops) *flops = 2.0 * n_dfma / (t * 1e-3);
    if (ms) *ms = t;
    return SF_OK;
}
