// gk_capi.cu -- the C ABI of include/gk_bfs.h.
//
// Every entry point catches failures and returns a gk_status with a
// thread-local message; nothing throws across the boundary.  There is no
// CPU path: without a device, compute entry points fail with
// GK_ERR_NO_DEVICE.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "gk_internal.cuh"

namespace {

// NVTX ranges name the host-side phases (graph build, trial, batch, Brandes)
// in nsys / ncu timelines; header-only, inert unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

thread_local std::string g_last_error;

gk_status fail(gk_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

gk_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return fail(GK_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return fail(GK_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
  return fail(GK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                       \
  do {                                       \
    cudaError_t e_ = (call);                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

gk_status need_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(GK_ERR_NO_DEVICE, "no CUDA device available (libgk_bfs has no CPU fallback)");
  if (device < 0 || device >= n) return fail(GK_ERR_INVALID, "device index out of range");
  CK(cudaSetDevice(device), "cudaSetDevice");
  return GK_OK;
}

void free_graph(gk_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->stream) {
    if (g->parent) cudaFreeAsync(g->parent, g->stream);
    cudaStreamSynchronize(g->stream);
  }
  if (g->in_off && g->in_off != g->out_off) cudaFree(g->in_off);
  if (g->in_nb && g->in_nb != g->out_nb) cudaFree(g->in_nb);
  cudaFree(g->out_off);
  cudaFree(g->out_nb);
  cudaFree(g->dead);
  cudaFree(g->off32);
  cudaFree(g->depth);
  cudaFree(g->acc);
  if (g->pool) cudaMemPoolDestroy(g->pool);
  if (g->batch_err) cudaFreeHost(g->batch_err);
  if (g->cm_peek) cudaFreeHost(g->cm_peek);
  for (cudaEvent_t e : g->batch_ev) cudaEventDestroy(e);
  for (int k = 0; k < 2; k++) {
    if (g->pk_dev[k]) cudaFree(g->pk_dev[k]);
    if (g->pk_host[k]) cudaFreeHost(g->pk_host[k]);
    if (g->pk_sc[k]) cudaEventDestroy(g->pk_sc[k]);
    if (g->pk_cp[k]) cudaEventDestroy(g->pk_cp[k]);
  }
  if (g->pk_cnt) cudaFree(g->pk_cnt);
  if (g->pk_total) cudaFreeHost(g->pk_total);
  if (g->pk_ev) cudaEventDestroy(g->pk_ev);
  if (g->sg_exec) cudaGraphExecDestroy(g->sg_exec);
  if (g->sg_graph) cudaGraphDestroy(g->sg_graph);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->stream) cudaStreamDestroy(g->stream);
  if (g->cstream) cudaStreamDestroy(g->cstream);
  if (g->stage) cudaFreeHost(g->stage);
  for (cudaEvent_t e : g->stage_ev) cudaEventDestroy(e);
  if (g->cstream2) cudaStreamDestroy(g->cstream2);
  if (g->cs2_done) cudaEventDestroy(g->cs2_done);
  delete g;
}

constexpr size_t kAlign = 256;
size_t up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }
size_t bitmap_bytes(int64_t n) { return up((size_t)((n + 31) / 32) * 4 + 64); }

// Graph-lifetime state: the dead-vertex layout (shared by BFS and Brandes),
// the launch geometry, streams/events and the per-trial memory pool.  No
// traversal-specific structure is derived from the graph here: every
// traversal builds its own scratch inside its timed region.
gk_status setup_graph(gk_graph* g, bool sorted) {
  const int64_t n = g->n;
  const int64_t w32 = (n + 31) / 32;
  CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking), "stream");
  CK(cudaEventCreate(&g->ev0), "event");
  CK(cudaEventCreate(&g->ev1), "event");
  CK(cudaMalloc(&g->acc, sizeof(unsigned long long) * 8), "alloc acc");
  CK(gk::bfs_configure(g->device, &g->launch), "configure bfs kernel");
  if (const char* fg = getenv("GK_L2_FETCH")) {  // A/B: the L2's maximum fetch granularity (bytes)
    size_t before = 0, after = 0;
    cudaDeviceGetLimit(&before, cudaLimitMaxL2FetchGranularity);
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(fg));
    cudaDeviceGetLimit(&after, cudaLimitMaxL2FetchGranularity);
    fprintf(stderr, "L2 fetch granularity %zu -> %zu\n", before, after);
    cudaGetLastError();
  }
  if (getenv("GK_NO_FRONT_SMEM")) g->launch.smem_front_max = 0;  // tests: large-graph paths on small graphs
  // Cluster mode for chains of tiny top-down levels.  gk_bfs reads the
  // hand-off state with the control block it reads anyway; gk_bfs_batch
  // pays a host round trip per trial for it, so it checks only on sparse
  // graphs (mean degree <= 8: road networks, meshes), where chains occur.
  CK(gk::cluster_configure(g->device, &g->cm_cluster, &g->cm_max_scout), "configure cluster kernel");
  if (g->cm_cluster) {
    CK(cudaHostAlloc(&g->cm_peek, sizeof(gk::Ctrl), cudaHostAllocDefault), "cudaHostAlloc");
    g->cm_batch = g->m <= 8 * g->n;
  }
  // Small graphs (n <= 8192 x cluster CTAs): one cluster runs the whole
  // traversal with its bitmaps in shared memory (gk_bfs_small.cu).
  CK(gk::small_configure(g->device, n, g->m, &g->small_cluster), "configure small-graph kernel");
  g->canary = getenv("GK_CANARY") && atoi(getenv("GK_CANARY")) != 0;
  CK(cudaMalloc(&g->dead, bitmap_bytes(n)), "alloc dead-vertex bitmap");
  CK(gk::dead_bitmap(g->in_off, n, g->dead, &g->live, g->stream), "dead-vertex bitmap");
  // The offsets' compact form (graph layout read by the BFS and Brandes
  // kernels, built with the graph like the dead bitmap): 4 bytes per vertex
  // instead of 8 on every offset read; undirected graphs up to 2^28
  // vertices (memory headroom at 2^30) and 2^33 arcs (one carry bit).
  if (!g->directed && n <= (int64_t(1) << 28) && g->m < (int64_t(2) << 32) && !getenv("GK_NO_OFF32")) {
    const int nhi = (int)(g->m >> 32);  // 0 or 1
    uint32_t* hi = nullptr;
    CK(cudaMalloc(&g->off32, sizeof(uint32_t) * (size_t)(n + 1) + 64), "alloc compact offsets");
    CK(cudaMalloc(&hi, sizeof(g->off_hi)), "alloc compact offsets");
    CK(cudaMemsetAsync(hi, 0xFF, sizeof(g->off_hi), g->stream), "compact offsets");
    cudaError_t e = gk::compact_offsets(g->out_off, n, g->off32, hi, nhi, g->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->off_hi, hi, sizeof(g->off_hi), cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    cudaFree(hi);
    CK(e, "compact offsets");
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = g->device;
  CK(cudaMemPoolCreate(&g->pool, &props), "memory pool");
  uint64_t keep = UINT64_MAX;  // keep freed blocks for the next trial
  CK(cudaMemPoolSetAttribute(g->pool, cudaMemPoolAttrReleaseThreshold, &keep), "memory pool");
  g->chunk_cap = 2 * (g->m / 1024) + 65536;  // >= 4 x warps when chunks shrink to 128 edges
  g->step_cap = std::min<int64_t>(n + 2, int64_t(1) << 20);
  // Owned-range hub expansion (gk_internal.cuh OwnEnt): one target range per
  // CTA of the launch, its slice of the next bitmap in dynamic shared memory
  // without lowering the occupancy; hubs = out-degree >= 32768 (with the
  // in-trial run search: 8192 -1%, 65536 same, 262144 -5% on kron27).  Off when the slice does not fit
  // (n > ~2^27 at 296 CTAs) or a list is not ascending (the per-range runs
  // are found by search).
  {
    const int r = g->launch.grid;
    const int64_t span_w = ((w32 + r - 1) / r + 3) & ~int64_t(3);
    const bool fits = (size_t)span_w * 4 <= g->launch.smem_keep_occ && (size_t)w32 * 4 > g->launch.smem_front_max;
    if (fits && sorted && !getenv("GK_NO_OWN")) {
      const char* dm = getenv("GK_OWN_DMIN");  // tests: hubs on small graphs
      g->own_dmin = dm ? std::max<int64_t>(1, strtoll(dm, nullptr, 10)) : 32768;
      int wl = 0;
      while ((int64_t(2) << wl) <= span_w) wl++;
      const int64_t nwin = (32 * span_w + (int64_t(1) << wl) - 1) >> wl;  // <= kOwnWin
      g->own_win_log = wl;
      g->own_r = r;
      g->own_span_w = span_w;
      g->own_cap = g->m / g->own_dmin + 1;  // hubs of one frontier, at most
      g->own_stage_bytes = sizeof(uint2) * (size_t)r * (size_t)(nwin << wl);
    }
  }
  CK(cudaStreamSynchronize(g->stream), "graph setup");
  return GK_OK;
}

// Per-trial scratch: one pool block for the traversal state (freed when the
// kernel is done), one for the bookkeeping read back afterwards (control
// block, step log), and the parent array (the result, kept until the next
// trial on this handle replaces it).
struct TrialBlocks {
  void* work = nullptr;
  void* book = nullptr;
  std::vector<std::pair<char*, const char*>> canaries;  // GK_CANARY: guard zones after each buffer
};
constexpr size_t kCanaryBytes = 4096;
constexpr unsigned char kCanaryByte = 0xA5;

// Carves consecutive buffers out of one pool block; in canary mode
// (GK_CANARY=1, a debug aid standing in for compute-sanitizer's memcheck,
// which this pool does not offer) every buffer is followed by a guard zone
// that trial_check_canaries verifies untouched after the kernel.
struct Carver {
  char* base;
  size_t at = 0;
  size_t cz;
  TrialBlocks* tb;
  char* take(size_t sz, const char* name) {
    char* r = base + at;
    at += sz;
    if (cz) {
      tb->canaries.emplace_back(base + at, name);
      at += cz;
    }
    return r;
  }
};

void carve_work(gk_graph* g, gk_trial* t, TrialBlocks* tb, size_t cz, size_t wb, size_t sz_q, size_t sz_ch,
                size_t sz_ol, size_t sz_os, bool own);

cudaError_t trial_alloc(gk_graph* g, gk_trial* t, TrialBlocks* tb, cudaStream_t s, bool own, bool small = false) {
  const size_t cz = g->canary ? kCanaryBytes : 0;
  const size_t wb = bitmap_bytes(g->n);
  const size_t sz_par = up(sizeof(int32_t) * std::max<int64_t>(g->n, 4) + 16);
  const size_t sz_q = up(sizeof(uint32_t) * (g->n + 1)), sz_ch = up(sizeof(gk::Chunk) * g->chunk_cap),
               sz_ol = own ? up(sizeof(gk::OwnEnt) * g->own_cap) : 0, sz_os = own ? up(g->own_stage_bytes) : 0;
  const size_t sz_ctrl = up(sizeof(gk::Ctrl)), sz_steps = up(sizeof(gk_step) * g->step_cap);
  const size_t work = 3 * (wb + cz) + sz_q + sz_ch + sz_ol + sz_os + (own ? 4 : 2) * cz;
  cudaError_t e;
  // The small-graph kernel needs no device scratch (its bitmaps and lists
  // live in shared memory): ONE pool block holds the result and the
  // bookkeeping, which then lives as long as the result.
  const size_t sz_book = sz_ctrl + sz_steps + 2 * cz;
  if ((e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&t->parent), sz_par + cz + (small ? sz_book : 0), g->pool,
                                   s)))
    return e;
  if (cz) tb->canaries.emplace_back(reinterpret_cast<char*>(t->parent) + sz_par, "parent");
  // the small-graph kernel keeps its bitmaps and lists in shared memory: no
  // scratch block.  (Order of the blocks: result, scratch, bookkeeping --
  // gk_bfs_batch's overlapped trials reuse the pool's blocks in that order;
  // allocating the small bookkeeping block second fragmented the pool and
  // cost the batch a third of its rate.)
  if (!small) {
    if ((e = cudaMallocFromPoolAsync(&tb->work, work, g->pool, s))) return e;
    carve_work(g, t, tb, cz, wb, sz_q, sz_ch, sz_ol, sz_os, own);
  }
  if (small) tb->book = nullptr;
  else if ((e = cudaMallocFromPoolAsync(&tb->book, sz_book, g->pool, s))) return e;
  Carver b{small ? reinterpret_cast<char*>(t->parent) + sz_par + cz : static_cast<char*>(tb->book), 0, cz, tb};
  t->ctrl = reinterpret_cast<gk::Ctrl*>(b.take(sz_ctrl, "ctrl"));
  t->steps = reinterpret_cast<gk_step*>(b.take(sz_steps, "steps"));
  for (auto& c : tb->canaries)
    if ((e = cudaMemsetAsync(c.first, kCanaryByte, cz, s))) return e;
  return cudaSuccess;
}

void carve_work(gk_graph* g, gk_trial* t, TrialBlocks* tb, size_t cz, size_t wb, size_t sz_q, size_t sz_ch,
                size_t sz_ol, size_t sz_os, bool own) {
  Carver w{static_cast<char*>(tb->work), 0, cz, tb};
  t->bits = reinterpret_cast<uint32_t*>(w.take(wb, "visited"));
  w.take(wb, "bm0");
  w.take(wb, "bm1");
  t->bits_stride = (wb + cz) / 4;
  t->queue = reinterpret_cast<uint32_t*>(w.take(sz_q, "queue"));
  t->chunks = reinterpret_cast<gk::Chunk*>(w.take(sz_ch, "chunks"));
  t->own_list = own ? reinterpret_cast<gk::OwnEnt*>(w.take(sz_ol, "own_list")) : nullptr;
  t->own_stage = own ? reinterpret_cast<uint2*>(w.take(sz_os, "own_stage")) : nullptr;
}

// GK_CANARY: every guard zone still holds its fill byte (call after the
// kernel, before the scratch is freed).
gk_status trial_check_canaries(gk_graph* g, const TrialBlocks& tb, cudaStream_t s) {
  for (const auto& c : tb.canaries) {
    unsigned long long bad = 0;
    CK(gk::canary_count(c.first, kCanaryBytes, kCanaryByte, g->acc, s), "canary check");
    CK(cudaMemcpyAsync(&bad, g->acc, sizeof(bad), cudaMemcpyDeviceToHost, s), "canary check");
    CK(cudaStreamSynchronize(s), "canary check");
    if (bad) return fail(GK_ERR_CUDA, std::string("canary zone after '") + c.second + "' overwritten (" +
                                          std::to_string(bad) + " bytes)");
  }
  return GK_OK;
}

void set_compact_offsets(const gk_graph* g, gk::BfsParams& p) {
  p.off32 = g->off32;
  p.off_hi[0] = g->off_hi[0];
}

// The trial's buffers in the kernel parameters (after trial_alloc).
void set_trial_ptrs(const gk_graph* g, const gk_trial& t, gk::BfsParams& p) {
  p.parent = t.parent;
  const size_t ww = t.bits_stride;
  p.visited = t.bits;
  p.bm0 = t.bits ? t.bits + ww : nullptr;
  p.bm1 = t.bits ? t.bits + 2 * ww : nullptr;
  p.queue = t.queue;
  p.chunks = t.chunks;
  p.ctrl = t.ctrl;
  p.steps = t.steps;
  if (t.own_list && !p.front_in_smem) {
    p.own_list = t.own_list;
    p.own_cap = g->own_cap;
    p.own_stage = t.own_stage;
    p.own_r = g->own_r;
    p.own_span_w = (int32_t)g->own_span_w;
    p.own_win_log = g->own_win_log;
    p.own_dmin = g->own_dmin;
  } else {
    p.own_list = nullptr;
  }
}

// Kernel parameters of one traversal on g (tuning knobs read from the environment).
gk::BfsParams make_params(gk_graph* g, const gk_trial& t, uint32_t source, int64_t alpha, int64_t beta,
                          int32_t strategy, int want_depth) {
  gk::BfsParams p{};
  p.n = g->n;
  p.m = g->m;
  p.w32 = (g->n + 31) / 32;
  p.out_off = g->out_off;
  p.out_nb = g->out_nb;
  p.in_off = g->in_off;
  p.in_nb = g->in_nb;
  p.src = source;
  p.strategy = strategy;
  p.alpha = alpha;
  p.beta = beta;
  p.want_depth = want_depth;
  p.front_in_smem = ((size_t)p.w32 * 4 <= g->launch.smem_front_max) ? 1 : 0;
  p.depth = g->depth;
  p.dead = g->dead;
  p.live = g->live;
  set_compact_offsets(g, p);
  set_trial_ptrs(g, t, p);
  // Large top-down steps additionally clear and fill the n/8-byte next
  // bitmap and sum degrees in a separate pass; worth it above ~n/16 edges.
  p.bitmap_td_min = std::max<int64_t>(4096, g->n / 16);
  // Range passes keep each pass's slice of the next bitmap within ~64 MB of
  // L2 (126 MB total; the rest holds visited lines, parent lines and the
  // stream).  Measured at kron30 (128 MB bitmap): 1 pass 27.8/34.8 ms,
  // 2 passes 23.0/27.5, 4 passes 25.8/32.5, 8 passes 29.5/38.7.
  {
    const int64_t budget = int64_t(64) << 20;
    int64_t passes = (p.w32 * 4 + budget - 1) / budget;
    if (const char* tp = getenv("GK_TD_PASSES")) passes = std::max<int64_t>(1, strtoll(tp, nullptr, 10));
    p.td_passes = (int32_t)std::max<int64_t>(1, passes);
    p.td_span = ((g->n + p.td_passes - 1) / p.td_passes + 31) / 32 * 32;
  }
  if (const char* bt = getenv("GK_BITMAP_TD_MIN")) p.bitmap_td_min = strtoll(bt, nullptr, 10);
  p.bu_tw_log_max = 5;
  p.w_lo = 0;  // one rank owns every word
  p.w_hi = p.w32;
  if (const char* tw = getenv("GK_BU_TASK_LOG")) p.bu_tw_log_max = std::max(0, std::min(5, atoi(tw)));
  // kTopDownRescan re-reads every new frontier's queue (bfs.hpp:161-167):
  // its steps keep the queue path (large steps leave the frontier a bitmap)
  if (strategy == GK_BFS_TOP_DOWN_RESCAN) p.bitmap_td_min = INT64_MAX;
  p.chunk_cap = g->chunk_cap;
  p.step_cap = g->step_cap;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  if (const char* w = getenv("GK_WATCHDOG_MS")) p.timeout_ns = strtoull(w, nullptr, 10) * 1000000ull;
  p.stop_after = 0xffffffffu;
  if (const char* sa = getenv("GK_STOP_AFTER")) p.stop_after = (unsigned)strtoul(sa, nullptr, 10);
  p.cm_ok = g->cm_cluster > 0;
  p.cm_max_scout = g->cm_max_scout;
  return p;
}

// The single-cluster kernel for this graph (GK_NO_SMALL=1: the grid kernel
// instead -- tests run both on the same small graphs).
bool use_small(const gk_graph* g) { return g->small_cluster > 0 && !getenv("GK_NO_SMALL"); }

bool use_own(const gk_graph* g) {
  return g->own_r > 0 && (size_t)((g->n + 31) / 32) * 4 > g->launch.smem_front_max;
}

gk_status kernel_error(const gk::Ctrl& ctrl, const char* what) {
  if (ctrl.error == 2) {
    unsigned lo = ~0u, hi = 0;
    for (int i = 0; i < 2048; i++) {
      if (ctrl.cta_ph[i] == 0) continue;
      lo = std::min(lo, ctrl.cta_ph[i]);
      hi = std::max(hi, ctrl.cta_ph[i]);
    }
    char buf[256];
    snprintf(buf, sizeof(buf),
             "%s kernel watchdog fired (grid barrier timeout): CTA barrier counts min %u max %u, arrivals %llu",
             what, lo, hi, (unsigned long long)ctrl.bar_count);
    return fail(GK_ERR_TIMEOUT, buf);
  }
  return fail(GK_ERR_CUDA, std::string(what) + " kernel: scratch buffer overflow");
}

// Cluster-mode hand-offs (gk_bfs_cluster.cu): after the grid kernel of a
// traversal handed off (h.mode != 0), runs whichever kernel the control
// block names next until the traversal has finished.  Each hand-off costs a
// host round trip (the next kernel is chosen here); a chain enters cluster
// mode only after kCmEnter tiny levels, so the trips are few.  Stops early
// on a kernel error, which the caller reads from the control block.
cudaError_t run_handoffs(gk_graph* g, gk::BfsParams p, cudaStream_t s, gk::Hand h) {
  while (h.mode != 0) {
    cudaError_t e;
    if (h.mode == 1) {
      e = gk::cluster_launch(p, h, g->cm_cluster, s);
    } else {
      p.resume = 1;
      p.rs = h;
      e = gk::bfs_launch(p, g->launch, s);
    }
    g->launches++;
    if (e != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(g->cm_peek, p.ctrl, gk::kCtrlPeek, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if (g->cm_peek->error) return cudaSuccess;
    h = g->cm_peek->hand;
#ifdef GK_CM_DEBUG
    {
      static auto t00 = std::chrono::steady_clock::now();
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t00).count();
      fprintf(stderr, "%.3f handoff: mode %lld nsteps %lld qs %lld qe %lld\n", ms, h.mode, h.nsteps, h.qs, h.qe);
    }
#endif
  }
  return cudaSuccess;
}

// The small-graph trial as a CUDA graph: [pool allocation of result +
// bookkeeping] -> [bfs_small].  Captured once per handle; the result's
// address is the graph's (freed by the next trial before the relaunch).
// Returns false when it cannot be built (the stream path runs instead).
bool small_graph_ready(gk_graph* g, const gk::BfsParams& p, cudaStream_t s) {
  if (g->sg_exec) return true;
  if (g->sg_failed) return false;
  g->sg_failed = true;
  gk_trial t;
  TrialBlocks tb;
  gk::BfsParams q = p;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaError_t e = trial_alloc(g, &t, &tb, s, false, true);
  if (e == cudaSuccess) {
    set_trial_ptrs(g, t, q);
    e = gk::small_launch(q, g->small_cluster, s);
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s, &graph);
  if (e != cudaSuccess || ec != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return false;
  }
  cudaGraphNode_t nodes[16];
  size_t nn = 16;
  cudaGraphNode_t kn = nullptr;
  if (cudaGraphGetNodes(graph, nodes, &nn) == cudaSuccess) {
    for (size_t i = 0; i < nn; i++) {
      cudaGraphNodeType ty;
      if (cudaGraphNodeGetType(nodes[i], &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) kn = nodes[i];
    }
  }
  cudaGraphExec_t exec = nullptr;
  if (!kn || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    cudaGraphDestroy(graph);
    cudaGetLastError();
    return false;
  }
  g->sg_graph = graph;
  g->sg_exec = exec;
  g->sg_kernel = kn;
  g->sg_trial = t;
  g->sg_failed = false;
  return true;
}

gk_status finish_graph(gk_graph* g, gk_graph** out) {
  if (g->n > (int64_t(1) << 31)) {  // every construction path: parents and depths are int32
    free_graph(g);
    return fail(GK_ERR_INVALID, "invalid graph: more than 2^31 vertices (parents are int32)");
  }
  // every kernel indexes with these arrays: reject a malformed CSR up front
  bool sorted = true;
  for (int pass = 0; pass < (g->directed ? 2 : 1); pass++) {
    bool off_ok = true, ids_ok = true, srt = true;
    const cudaError_t e = gk::validate_csr(pass ? g->in_off : g->out_off, pass ? g->in_nb : g->out_nb, g->n, g->m,
                                           g->n, &off_ok, &ids_ok, pass ? nullptr : &srt, nullptr);
    if (e != cudaSuccess || !off_ok || !ids_ok) {
      free_graph(g);
      if (e != cudaSuccess) return cuda_fail(e, "validate CSR");
      return fail(GK_ERR_INVALID, !off_ok ? "invalid graph: offsets not monotone from 0 to m"
                                          : "invalid graph: neighbour id out of range");
    }
    if (!pass) sorted = srt;
  }
  gk_status st = setup_graph(g, sorted);
  if (st != GK_OK) {
    free_graph(g);
    return st;
  }
  *out = g;
  return GK_OK;
}

}  // namespace

extern "C" {

const char* gk_last_error(void) { return g_last_error.c_str(); }
int gk_abi_version(void) { return GK_ABI_VERSION; }

int gk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

gk_status gk_graph_upload(const gk_csr_view* csr, int device, gk_graph** out) {
  NvtxRange nvtx_range("gk_graph_upload");
  if (!csr || !out || !csr->out_offsets || csr->num_nodes < 0)
    return fail(GK_ERR_INVALID, "gk_graph_upload: null argument");
  if (csr->num_nodes > (int64_t(1) << 31))
    return fail(GK_ERR_INVALID, "gk_graph_upload: more than 2^31 vertices (parents are int32)");
  if (csr->directed && (!csr->in_offsets || (!csr->in_neighbors && csr->out_offsets[csr->num_nodes])))
    return fail(GK_ERR_INVALID, "gk_graph_upload: directed graph needs in_* arrays");
  gk_status st = need_device(device);
  if (st != GK_OK) return st;
  auto* g = new gk_graph;
  g->device = device;
  g->n = csr->num_nodes;
  g->m = csr->out_offsets[csr->num_nodes];
  g->directed = csr->directed ? 1 : 0;
  const size_t ob = sizeof(int64_t) * (g->n + 1), nbb = sizeof(uint32_t) * std::max<int64_t>(g->m, 1);
  cudaError_t e;
  if ((e = cudaMalloc(&g->out_off, ob + 16)) || (e = cudaMalloc(&g->out_nb, nbb + gk::kNbPad)) ||
      (e = cudaMemcpy(g->out_off, csr->out_offsets, ob, cudaMemcpyHostToDevice)) ||
      (g->m && (e = cudaMemcpy(g->out_nb, csr->out_neighbors, sizeof(uint32_t) * g->m,
                               cudaMemcpyHostToDevice)))) {
    free_graph(g);
    return cuda_fail(e, "upload CSR");
  }
  if (g->directed) {
    if ((e = cudaMalloc(&g->in_off, ob + 16)) || (e = cudaMalloc(&g->in_nb, nbb + gk::kNbPad)) ||
        (e = cudaMemcpy(g->in_off, csr->in_offsets, ob, cudaMemcpyHostToDevice)) ||
        (g->m && (e = cudaMemcpy(g->in_nb, csr->in_neighbors, sizeof(uint32_t) * g->m,
                                 cudaMemcpyHostToDevice)))) {
      free_graph(g);
      return cuda_fail(e, "upload in-CSR");
    }
  } else {
    g->in_off = g->out_off;  // graph.hpp:64-67: in aliases out when undirected
    g->in_nb = g->out_nb;
  }
  return finish_graph(g, out);
}

gk_status gk_graph_generate(int kind, int scale, int degree, uint64_t seed, int permute,
                            int device, gk_graph** out) {
  NvtxRange nvtx_range("gk_graph_generate");
  if (!out) return fail(GK_ERR_INVALID, "gk_graph_generate: null out");
  if (kind != 0 && kind != 1) return fail(GK_ERR_INVALID, "generator kind must be 0 (kron) or 1 (urand)");
  if (scale < 1 || scale > 31) return fail(GK_ERR_INVALID, "generator scale must be in [1, 31]");
  if (degree < 1) return fail(GK_ERR_INVALID, "generator avg_degree must be >= 1");
  gk_status st = need_device(device);
  if (st != GK_OK) return st;
  gk::DevCsr csr;
  std::string err;
  cudaError_t e = gk::build_generated(kind, scale, degree, seed, permute, 0, -1, &csr, &err);
  if (e != cudaSuccess) return cuda_fail(e, err.empty() ? "device graph build" : err.c_str());
  auto* g = new gk_graph;
  g->device = device;
  g->n = csr.n;
  g->m = csr.m;
  g->out_off = g->in_off = csr.off;
  g->out_nb = g->in_nb = csr.nb;
  return finish_graph(g, out);
}

gk_status gk_graph_generate_grid(int64_t rows, int64_t cols, double p_delete, double p_diag,
                                 uint64_t seed, int device, gk_graph** out) {
  NvtxRange nvtx_range("gk_graph_generate_grid");
  if (!out) return fail(GK_ERR_INVALID, "gk_graph_generate_grid: null out");
  if (rows < 1 || cols < 1 || rows * cols > (int64_t(1) << 31))
    return fail(GK_ERR_INVALID, "grid dimensions out of range");
  if (!(p_delete >= 0 && p_delete <= 1 && p_diag >= 0 && p_diag <= 1))
    return fail(GK_ERR_INVALID, "grid probabilities must be in [0, 1]");
  gk_status st = need_device(device);
  if (st != GK_OK) return st;
  gk::DevCsr csr;
  std::string err;
  cudaError_t e = gk::build_grid(rows, cols, p_delete, p_diag, seed, &csr, &err);
  if (e != cudaSuccess) return cuda_fail(e, err.empty() ? "device grid build" : err.c_str());
  auto* g = new gk_graph;
  g->device = device;
  g->n = csr.n;
  g->m = csr.m;
  g->out_off = g->in_off = csr.off;
  g->out_nb = g->in_nb = csr.nb;
  return finish_graph(g, out);
}

gk_status gk_graph_load_sg(const char* path, int device, gk_graph** out) {
  NvtxRange nvtx_range("gk_graph_load_sg");
  if (!path || !out) return fail(GK_ERR_INVALID, "gk_graph_load_sg: null argument");
  gk_status st = need_device(device);
  if (st != GK_OK) return st;
  auto* g = new gk_graph;
  g->device = device;
  std::string err;
  int64_t n = 0, m = 0;
  int directed = 0;
  const int code = gk::sg_load(path, &n, &m, &directed, &g->out_off, &g->out_nb, &g->in_off, &g->in_nb, &err);
  if (code) {
    delete g;
    if (code == 7 || code == 8) return fail(GK_ERR_OOM, err);
    if (code == 2) return fail(GK_ERR_INVALID, err);
    return fail(GK_ERR_LOAD, err);
  }
  g->n = n;
  g->m = m;
  g->directed = directed;
  if (!directed) {
    g->in_off = g->out_off;
    g->in_nb = g->out_nb;
  }
  return finish_graph(g, out);
}

gk_status gk_graph_save_sg(const gk_graph* g, const char* path) {
  if (!g || !path) return fail(GK_ERR_INVALID, "gk_graph_save_sg: null argument");
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  std::string err;
  const int code = gk::sg_save(path, g->n, g->m, g->directed, g->out_off, g->out_nb, g->in_off, g->in_nb, &err);
  if (code) return fail(code == 2 ? GK_ERR_INVALID : GK_ERR_LOAD, err);
  return GK_OK;
}

void gk_graph_free(gk_graph* g) { free_graph(g); }

gk_status gk_graph_info(const gk_graph* g, int64_t* n, int64_t* m, int32_t* directed) {
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (directed) *directed = g->directed;
  return GK_OK;
}

gk_status gk_graph_download(const gk_graph* g, int64_t* out_offsets, uint32_t* out_neighbors,
                            int64_t* in_offsets, uint32_t* in_neighbors) {
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  const size_t ob = sizeof(int64_t) * (g->n + 1), nbb = sizeof(uint32_t) * g->m;
  if (out_offsets) CK(cudaMemcpy(out_offsets, g->out_off, ob, cudaMemcpyDeviceToHost), "download");
  if (out_neighbors && g->m) CK(cudaMemcpy(out_neighbors, g->out_nb, nbb, cudaMemcpyDeviceToHost), "download");
  if (in_offsets) CK(cudaMemcpy(in_offsets, g->in_off, ob, cudaMemcpyDeviceToHost), "download");
  if (in_neighbors && g->m) CK(cudaMemcpy(in_neighbors, g->in_nb, nbb, cudaMemcpyDeviceToHost), "download");
  return GK_OK;
}

// source_picker.hpp:22-54: Rng(seed) draws NextBounded(n), rejecting
// zero out-degree candidates; degrees are read from the device offsets.
gk_status gk_pick_sources(const gk_graph* g, int64_t count, uint64_t seed, uint32_t* out) {
  if (!g || (!out && count > 0)) return fail(GK_ERR_INVALID, "null argument");
  if (g->m == 0) return fail(GK_ERR_NO_EDGES, "cannot pick sources: graph has no edges");
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  auto mix = [](uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  };
  uint64_t state = mix(seed) ^ mix(~0ULL);
  auto next = [&]() {
    state += 0x9e3779b97f4a7c15ULL;
    return mix(state - 0x9e3779b97f4a7c15ULL);
  };
  const uint32_t bound = (uint32_t)g->n;
  uint32_t mask = bound - 1;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  for (int64_t i = 0; i < count; i++) {
    for (;;) {
      uint32_t c;
      do {
        c = (uint32_t)(next() >> 32) & mask;
      } while (c >= bound);
      int64_t o[2];
      CK(cudaMemcpy(o, g->out_off + c, sizeof(o), cudaMemcpyDeviceToHost), "read degree");
      if (o[1] != o[0]) {
        out[i] = c;
        break;
      }
    }
  }
  return GK_OK;
}

gk_status gk_bfs_keep_depth(gk_graph* g, int32_t keep) {
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  g->keep_depth = keep ? 1 : 0;
  return GK_OK;
}

// A result copied into caller memory.  Pinned destinations (and small
// copies) take one cudaMemcpyAsync.  Pageable ones would go through the
// driver's own staging at ~16 GB/s on the GPU box (tools/bench_mem/
// hostcopy.cu); instead the array moves in 16 MiB chunks into a pinned
// stage kept with the graph (~55 GB/s), and host threads copy each chunk out
// as soon as its event fires, overlapping the next chunks' transfers.
// Synchronous: the data is in `dst` on return.
static cudaError_t copy_out(gk_graph* g, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  static const bool no_stage = getenv("GK_NO_STAGE") != nullptr;  // A/B switch
  constexpr size_t kChunk = size_t(16) << 20;
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type != cudaMemoryTypeUnregistered;
  cudaGetLastError();  // older drivers flag unregistered pointers
  cudaError_t e;
  if (pinned || no_stage || bytes < 2 * kChunk) {
    if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s))) return e;
    return cudaStreamSynchronize(s);
  }
  if (g->stage_bytes < bytes) {
    if (g->stage) cudaFreeHost(g->stage);
    g->stage = nullptr;
    g->stage_bytes = 0;
    if ((e = cudaHostAlloc(&g->stage, bytes, cudaHostAllocDefault))) return e;
    g->stage_bytes = bytes;
  }
  const size_t chunks = (bytes + kChunk - 1) / kChunk;
  while (g->stage_ev.size() < chunks) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return e;
    g->stage_ev.push_back(ev);
  }
  for (size_t k = 0; k < chunks; k++) {
    const size_t a = k * kChunk, len = std::min(kChunk, bytes - a);
    if ((e = cudaMemcpyAsync(g->stage + a, static_cast<const char*>(src) + a, len, cudaMemcpyDeviceToHost, s)))
      return e;
    if ((e = cudaEventRecord(g->stage_ev[k], s))) return e;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  const int nt = (int)std::max(1u, std::min(16u, hw ? hw : 1u));
  std::vector<cudaError_t> errs(nt, cudaSuccess);
  auto work = [&](int t) {
    cudaSetDevice(g->device);
    for (size_t k = 0; k < chunks; k++) {
      if (cudaError_t ee = cudaEventSynchronize(g->stage_ev[k])) {
        errs[t] = ee;
        return;
      }
      const size_t a = k * kChunk, len = std::min(kChunk, bytes - a);
      const size_t lo = a + len * t / nt, hi = a + len * (t + 1) / nt;
      memcpy(static_cast<char*>(dst) + lo, g->stage + lo, hi - lo);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; t++) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (cudaError_t ee : errs)
    if (ee) return ee;
  return cudaSuccess;
}

gk_status gk_bfs(gk_graph* g, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy,
                 int32_t* parent_out, int32_t* depth_out, gk_bfs_stats* stats) {
  NvtxRange nvtx_range("gk_bfs");
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  // bfs.hpp:120-123, same order and messages
  if ((int64_t)source >= g->n) return fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  if (alpha <= 0 || beta <= 0) return fail(GK_ERR_BAD_PARAM, "bfs alpha and beta must be positive");
  if (strategy < 0 || strategy > 2) return fail(GK_ERR_BAD_PARAM, "unknown bfs strategy");
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  const int want_depth = (depth_out != nullptr) || g->keep_depth;
  if (want_depth && !g->depth)
    CK(cudaMalloc(&g->depth, sizeof(int32_t) * std::max<int64_t>(g->n, 4) + 16), "alloc depth");
  cudaStream_t s = g->stream;
  g->last_valid = 0;
  if (g->parent) {  // the previous result goes back to the pool
    CK(cudaFreeAsync(g->parent, s), "free previous result");
    g->parent = nullptr;
  }
  // Timed trial: allocation of the result and every scratch buffer, their
  // initialisation, the traversal, the release of the scratch.
  gk_trial t;
  TrialBlocks tb;
  const bool small = use_small(g);
  // kernel arguments (host work, the environment's tuning switches) ahead of
  // the trial; the trial's own buffers are filled in after its allocation
  gk::BfsParams p = make_params(g, t, source, alpha, beta, strategy, want_depth);
  static const bool host_timing = getenv("GK_HOST_TIMING") != nullptr;  // diagnostics
  // small graphs: the trial is one CUDA graph launch (allocation node +
  // kernel); its arguments are set here, before the timed region
  const bool as_graph = small && !g->canary && !getenv("GK_NO_SMALL_GRAPH") && small_graph_ready(g, p, s);
  if (as_graph) {
    set_trial_ptrs(g, g->sg_trial, p);
    cudaKernelNodeParams kp{};
    CK(cudaGraphKernelNodeGetParams(g->sg_kernel, &kp), "small-graph kernel node");
    void* args[] = {&p};
    kp.kernelParams = args;
    kp.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(g->sg_exec, g->sg_kernel, &kp), "small-graph kernel arguments");
  }
  const auto h0 = std::chrono::steady_clock::now();
  CK(cudaEventRecord(g->ev0, s), "event record");
  const auto h1 = std::chrono::steady_clock::now();
  if (as_graph) {
    t = g->sg_trial;
  } else {
    CK(trial_alloc(g, &t, &tb, s, !small && use_own(g), small), "allocate trial scratch");
    set_trial_ptrs(g, t, p);
  }
  g->parent = t.parent;
  const auto h2 = std::chrono::steady_clock::now();
  if (as_graph) CK(cudaGraphLaunch(g->sg_exec, s), "launch small-graph trial");
  else if (small) CK(gk::small_launch(p, g->small_cluster, s), "launch small-graph bfs kernel");
  else CK(gk::bfs_launch(p, g->launch, s), "launch bfs kernel");
  g->launches++;
  const auto h3 = std::chrono::steady_clock::now();
  CK(cudaEventRecord(g->ev1, s), "event record");
  if (host_timing) {
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "gk_bfs host: record ev0 %.1f us, alloc %.1f us, launch %.1f us\n", us(h0, h1), us(h1, h2),
            us(h2, h3));
  }
  gk::Ctrl& ctrl = g->last_ctrl;
  CK(cudaMemcpyAsync(&ctrl, t.ctrl, sizeof(ctrl), cudaMemcpyDeviceToHost, s), "read ctrl");
  CK(cudaStreamSynchronize(s), "bfs kernel");
  if (!ctrl.error && ctrl.hand.mode != 0) {  // the grid kernel handed off to the cluster kernel
    CK(run_handoffs(g, p, s, ctrl.hand), "cluster-mode hand-off");
    CK(cudaEventRecord(g->ev1, s), "event record");
    CK(cudaMemcpyAsync(&ctrl, t.ctrl, sizeof(ctrl), cudaMemcpyDeviceToHost, s), "read ctrl");
    CK(cudaStreamSynchronize(s), "bfs kernel");
  }
  if (g->canary) {
    const gk_status cst = trial_check_canaries(g, tb, s);
    if (cst != GK_OK) return cst;
  }
  // the scratch returns to the pool (stream-ordered bookkeeping, no device work)
  if (tb.work) CK(cudaFreeAsync(tb.work, s), "free trial scratch");
  if (ctrl.error) {
    if (tb.book) cudaFreeAsync(tb.book, s);
    return kernel_error(ctrl, "bfs");
  }
  g->last_valid = 1;
  g->depth_valid = want_depth;
  gk_status st = GK_OK;
  if (stats) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1), "event time");
    stats->device_ms = ms;
    stats->num_steps = (int32_t)ctrl.num_steps;
    if (stats->steps && stats->max_steps > 0) {
      int64_t k = std::min<int64_t>({(int64_t)stats->max_steps, ctrl.num_steps, g->step_cap});
      if (k > 0)
        CK(cudaMemcpyAsync(stats->steps, t.steps, sizeof(gk_step) * k, cudaMemcpyDeviceToHost, s), "read steps");
    }
    if (stats->want_counts) {
      CK(gk::count_reached(g->parent, g->out_off, g->n, g->acc, s), "count reached");
      unsigned long long two[2];
      CK(cudaMemcpyAsync(two, g->acc, sizeof(two), cudaMemcpyDeviceToHost, s), "read counts");
      CK(cudaStreamSynchronize(s), "count reached");
      stats->reached = (int64_t)two[0];
      stats->component_edges = (int64_t)(g->directed ? two[1] : two[1] / 2);
    }
  }
  if (tb.book) CK(cudaFreeAsync(tb.book, s), "free trial bookkeeping");
  if (parent_out && g->n) CK(copy_out(g, parent_out, g->parent, sizeof(int32_t) * g->n, s), "D2H parent");
  if (depth_out && g->n) CK(copy_out(g, depth_out, g->depth, sizeof(int32_t) * g->n, s), "D2H depth");
  CK(cudaStreamSynchronize(s), "D2H");
  return st;
}

// Many traversals with their parent arrays returned to host memory: the
// D2H copy of traversal i (on a second stream) overlaps traversal i+1, so a
// run is bound by max(kernel, copy) per source instead of their sum.  Every
// trial allocates its result and scratch from the pool inside its own
// timed region; a result returns to the pool once its copy has finished.
// Same validation and results as gk_bfs.
gk_status gk_bfs_batch(gk_graph* g, const uint32_t* sources, int32_t count, int64_t alpha, int64_t beta,
                       int32_t strategy, int32_t* const* parents_out, float* device_ms) {
  NvtxRange nvtx_range("gk_bfs_batch");
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  if (count < 0 || (count > 0 && !sources)) return fail(GK_ERR_INVALID, "null argument");
  for (int32_t i = 0; i < count; i++)
    if ((int64_t)sources[i] >= g->n) return fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  if (alpha <= 0 || beta <= 0) return fail(GK_ERR_BAD_PARAM, "bfs alpha and beta must be positive");
  if (strategy < 0 || strategy > 2) return fail(GK_ERR_BAD_PARAM, "unknown bfs strategy");
  if (count == 0) return GK_OK;
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  if (!g->cstream) CK(cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking), "stream");
  const bool split = getenv("GK_BATCH_SPLIT") && atoi(getenv("GK_BATCH_SPLIT")) != 0;
  if (split && !g->cstream2) {
    CK(cudaStreamCreateWithFlags(&g->cstream2, cudaStreamNonBlocking), "stream");
    CK(cudaEventCreateWithFlags(&g->cs2_done, cudaEventDisableTiming), "event");
  }
  const size_t nev = 3 * (size_t)count;  // per trial: start, end, copy done
  while (g->batch_ev.size() < nev) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e), "event create");
    g->batch_ev.push_back(e);
  }
  if (g->batch_err_cap < count) {
    if (g->batch_err) cudaFreeHost(g->batch_err);
    g->batch_err = nullptr;
    g->batch_err_cap = 0;
    CK(cudaHostAlloc(&g->batch_err, sizeof(int) * count, cudaHostAllocDefault), "cudaHostAlloc");
    g->batch_err_cap = count;
  }
  cudaStream_t s = g->stream, cs = g->cstream;
  cudaEvent_t* ev = g->batch_ev.data();
  int* errs = g->batch_err;
  g->last_valid = 0;
  g->depth_valid = 0;
  if (g->parent) {
    CK(cudaFreeAsync(g->parent, s), "free previous result");
    g->parent = nullptr;
  }
  const bool small = use_small(g);
  const bool own = !small && use_own(g);
  // Compact transfer of the results (gk_pack.cu) on graphs from 2^22
  // vertices; a source whose reached set makes it no smaller goes raw.
  static const char* pk_env = getenv("GK_BATCH_PACK");
  const bool pack = parents_out && g->n >= (int64_t(1) << 22) && !(pk_env && atoi(pk_env) == 0) && !split;
  const int64_t nblk = (g->n + 1023) / 1024;
  const size_t pk_bytes = sizeof(uint32_t) * gk::pack_words(g->n);
  if (pack && !g->pk_dev[0]) {
    for (int k = 0; k < 2; k++) {
      CK(cudaMalloc(&g->pk_dev[k], pk_bytes), "alloc transfer buffer");
      CK(cudaHostAlloc(&g->pk_host[k], pk_bytes, cudaHostAllocDefault), "cudaHostAlloc transfer stage");
      CK(cudaEventCreateWithFlags(&g->pk_sc[k], cudaEventDisableTiming), "event");
      CK(cudaEventCreateWithFlags(&g->pk_cp[k], cudaEventDisableTiming | cudaEventBlockingSync), "event");
    }
    CK(cudaMalloc(&g->pk_cnt, sizeof(uint32_t) * (nblk + 1)), "alloc block counts");
    CK(cudaHostAlloc(&g->pk_total, sizeof(uint32_t) * 2, cudaHostAllocDefault), "cudaHostAlloc");
    CK(cudaEventCreateWithFlags(&g->pk_ev, cudaEventDisableTiming | cudaEventBlockingSync), "event");
  }
  // GK_PACK_RAW_FRAC (A/B, default 0): blocks [0, raw_blk) travel raw
  // straight into the caller's array after the compact rest.  Measured on
  // kron27 (profiles/r02/e2e_compact_kron27.txt): raw shares 0 / 0.15 / 0.25
  // / 0.35 give 245 / 236 / 227 / 213 GTEPS -- the DMA writes and the host
  // expansion share the host's memory bandwidth, and DMA bytes cost more.
  static const double raw_frac = getenv("GK_PACK_RAW_FRAC") ? atof(getenv("GK_PACK_RAW_FRAC")) : 0.0;
  const int64_t raw_blk = std::min<int64_t>(nblk - 1, std::max<int64_t>(0, (int64_t)(raw_frac * nblk)));
  static const int exp_threads = getenv("GK_EXPAND_THREADS") ? atoi(getenv("GK_EXPAND_THREADS"))
                                                              : (int)std::thread::hardware_concurrency() - 1;
  std::thread expander[2];  // host expansion of source i runs in expander[i & 1]
  int exp_err[2] = {0, 0};
  int32_t* exp_dst[2] = {nullptr, nullptr};
  auto settle = [&](const int32_t* dst) {  // outputs may repeat: one writer per array at a time
    for (int k = 0; k < 2; k++)
      if (expander[k].joinable() && exp_dst[k] == dst) expander[k].join();
  };
  g->last_d2h_bytes = 0;
  g->last_packed = 0;
  cudaError_t e = cudaSuccess;
  if (!g->batch_warm && count > 1) {
    // Up to three trials' blocks are live at once here (a result is freed
    // only after its copy); grow the pool to that once, so no trial pays
    // for the pool's first mapping of the memory.
    gk_trial tw[3];
    TrialBlocks bw[3];
    int k = 0;
    for (; k < 3 && e == cudaSuccess; k++) e = trial_alloc(g, &tw[k], &bw[k], s, own, small);
    for (int j = 0; j < k; j++) {
      if (tw[j].parent) cudaFreeAsync(tw[j].parent, s);
      if (bw[j].work) cudaFreeAsync(bw[j].work, s);
      if (bw[j].book) cudaFreeAsync(bw[j].book, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(GK_ERR_CUDA, std::string("bfs batch: ") + cudaGetErrorString(e));
    g->batch_warm = true;
  }
  for (int32_t i = 0; i < count && e == cudaSuccess; i++) {
    gk_trial t;
    TrialBlocks tb;
    // the copy of trial i-2 has returned its result to the pool
    if (i >= 2 && (e = cudaStreamWaitEvent(s, ev[3 * (i - 2) + 2], 0))) break;
    if ((e = cudaEventRecord(ev[3 * i], s))) break;
    if ((e = trial_alloc(g, &t, &tb, s, own, small))) break;
    gk::BfsParams p = make_params(g, t, sources[i], alpha, beta, strategy, 0);
    p.cm_ok = g->cm_batch && !small ? p.cm_ok : 0;
    if ((e = small ? gk::small_launch(p, g->small_cluster, s) : gk::bfs_launch(p, g->launch, s))) break;
    g->launches++;
    if (p.cm_ok) {  // hand-offs are decided on the host: wait for the grid kernel
      if ((e = cudaMemcpyAsync(g->cm_peek, p.ctrl, gk::kCtrlPeek, cudaMemcpyDeviceToHost, s))) break;
#ifdef GK_CM_DEBUG
      static auto t00 = std::chrono::steady_clock::now();
      const double ms0 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t00).count();
#endif
      if ((e = cudaStreamSynchronize(s))) break;
#ifdef GK_CM_DEBUG
      const double ms1 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t00).count();
      fprintf(stderr, "trial %d: grid kernel enqueued %.3f synced %.3f mode %lld nsteps %lld\n", i, ms0, ms1,
              g->cm_peek->hand.mode, g->cm_peek->hand.nsteps);
#endif
      if (!g->cm_peek->error && g->cm_peek->hand.mode != 0 && (e = run_handoffs(g, p, s, g->cm_peek->hand))) break;
    }
    if (tb.work && (e = cudaFreeAsync(tb.work, s))) break;
    if ((e = cudaEventRecord(ev[3 * i + 1], s))) break;
    if ((e = cudaMemcpyAsync(errs + i, &t.ctrl->error, sizeof(int), cudaMemcpyDeviceToHost, s))) break;
    if (tb.book && (e = cudaFreeAsync(tb.book, s))) break;
    bool packed = false;
    if (pack && parents_out[i] && !g->pk_raw) {
      // the transfer buffer i & 1 is free: trial i waited for the copy of i - 2
      const int k = i & 1;
      // (the scan kernel can also store these two words into mapped pinned
      // memory, bypassing the copy engine: kron27 e2e fell to 54 GTEPS with
      // it -- the copies stay)
      if ((e = gk::pack_count(t.parent, g->n, g->pk_dev[k], g->pk_cnt, raw_blk, nullptr, s))) break;
      if ((e = cudaMemcpyAsync(g->pk_total, g->pk_dev[k] + nblk, sizeof(uint32_t), cudaMemcpyDeviceToHost, s))) break;
      if ((e = cudaMemcpyAsync(g->pk_total + 1, g->pk_dev[k] + raw_blk, sizeof(uint32_t), cudaMemcpyDeviceToHost, s)))
        break;
      if ((e = cudaEventRecord(g->pk_ev, s))) break;
      if ((e = cudaEventSynchronize(g->pk_ev))) break;  // trial i is done and its reached count known
      const size_t words = gk::pack_words(g->n) - (size_t)g->n + *g->pk_total;
      if (words >= (size_t)g->n) {
        // this graph's sources reach (nearly) everything: its later results
        // go raw without the count pass and its host round trip (urand27:
        // 62 GTEPS e2e with a count per source, 159 without)
        g->pk_raw = true;
      } else {
        packed = true;
        if ((e = gk::pack_scatter(t.parent, g->n, g->pk_dev[k], s))) break;
        if ((e = cudaEventRecord(g->pk_sc[k], s))) break;
        if (expander[k].joinable()) expander[k].join();  // stage k: source i - 2 expanded
        if (exp_err[k]) break;
        if ((e = cudaStreamWaitEvent(cs, g->pk_sc[k], 0))) break;
        // offsets + bitmap, then the compact part's packed parents (same
        // offsets in the stage), then the raw head into the caller's array
        const size_t head = (size_t)(nblk + 1 + 32 * nblk), skip = g->pk_total[1];
        if ((e = cudaMemcpyAsync(g->pk_host[k], g->pk_dev[k], sizeof(uint32_t) * head, cudaMemcpyDeviceToHost, cs)))
          break;
        if (words > head + skip &&
            (e = cudaMemcpyAsync(g->pk_host[k] + head + skip, g->pk_dev[k] + head + skip,
                                 sizeof(uint32_t) * (words - head - skip), cudaMemcpyDeviceToHost, cs)))
          break;
        if ((e = cudaEventRecord(g->pk_cp[k], cs))) break;
        if (raw_blk > 0 && (e = cudaMemcpyAsync(parents_out[i], t.parent, sizeof(int32_t) * 1024 * raw_blk,
                                                 cudaMemcpyDeviceToHost, cs)))
          break;
        g->last_d2h_bytes += (int64_t)(sizeof(uint32_t) * (words - skip) + sizeof(int32_t) * 1024 * raw_blk);
        g->last_packed++;
      }
    }
    if ((e = cudaStreamWaitEvent(cs, ev[3 * i + 1], 0))) break;
    if (packed) {
      // expanded by the host below, once this copy has landed
    } else if (parents_out && parents_out[i]) {
      settle(parents_out[i]);
      g->last_d2h_bytes += (int64_t)(sizeof(int32_t) * g->n);
      // GK_BATCH_SPLIT: the two halves on two copy streams (two DMA engines)
      const size_t bytes = sizeof(int32_t) * g->n, half = split ? (bytes / 2 + 255) & ~size_t(255) : bytes;
      if ((e = cudaMemcpyAsync(parents_out[i], t.parent, half, cudaMemcpyDeviceToHost, cs))) break;
      if (half < bytes) {
        if ((e = cudaStreamWaitEvent(g->cstream2, ev[3 * i + 1], 0))) break;
        if ((e = cudaMemcpyAsync(reinterpret_cast<char*>(parents_out[i]) + half, reinterpret_cast<char*>(t.parent) + half,
                                 bytes - half, cudaMemcpyDeviceToHost, g->cstream2)))
          break;
        if ((e = cudaEventRecord(g->cs2_done, g->cstream2))) break;
        if ((e = cudaStreamWaitEvent(cs, g->cs2_done, 0))) break;
      }
    }
    if (i + 1 < count) {
      if ((e = cudaFreeAsync(t.parent, cs))) break;
    } else {
      g->parent = t.parent;  // the last result stays for gk_bfs_device_parent
    }
    if ((e = cudaEventRecord(ev[3 * i + 2], cs))) break;
    if (packed) {
      const int k = i & 1;
      cudaEvent_t done = g->pk_cp[k];
      const int64_t first = raw_blk;
      int32_t* dst = parents_out[i];
      const uint32_t* stage = g->pk_host[k];
      const int64_t n = g->n;
      const int dev = g->device;
      int* err = &exp_err[k];
      settle(dst);
      exp_dst[k] = dst;
      expander[k] = std::thread([=]() {
        cudaSetDevice(dev);
        if (cudaEventSynchronize(done) != cudaSuccess) {
          *err = 1;
          return;
        }
        gk::expand_parents(stage, n, dst, exp_threads, first);
      });
    }
  }
  for (auto& th : expander)
    if (th.joinable()) th.join();
  if (e == cudaSuccess && (exp_err[0] || exp_err[1])) e = cudaErrorUnknown;
  if (g->cstream2) cudaStreamSynchronize(g->cstream2);
  cudaError_t e2 = cudaStreamSynchronize(s), e3 = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : e3;
  if (e != cudaSuccess) return fail(GK_ERR_CUDA, std::string("bfs batch: ") + cudaGetErrorString(e));
  for (int32_t i = 0; i < count; i++) {
    if (errs[i] == 2) return fail(GK_ERR_TIMEOUT, "bfs kernel watchdog fired (grid barrier timeout)");
    if (errs[i]) return fail(GK_ERR_CUDA, "bfs kernel: scratch buffer overflow");
    if (device_ms) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[3 * i], ev[3 * i + 1]);
      device_ms[i] = ms;
    }
  }
  return GK_OK;
}

int64_t gk_bfs_batch_d2h_bytes(const gk_graph* g, int64_t* packed) {
  if (packed) *packed = g ? g->last_packed : 0;
  return g ? g->last_d2h_bytes : 0;
}

const int32_t* gk_bfs_device_parent(const gk_graph* g) { return g ? g->parent : nullptr; }
int64_t gk_bfs_launches(const gk_graph* g) { return g ? (int64_t)g->launches : 0; }
int32_t* gk_bfs_device_depth(const gk_graph* g) { return g && g->depth_valid ? g->depth : nullptr; }

gk_status gk_bfs_trace(const gk_graph* g, uint64_t* ts_ns, char* tags, int32_t cap, int32_t* count) {
  if (!g || !count) return fail(GK_ERR_INVALID, "null argument");
  if (!g->last_valid) return fail(GK_ERR_INVALID, "no completed gk_bfs on this handle");
  // entries up to the first untagged one (diagnostic builds may tag entries
  // past a gap: GK_TRACE_ALL=1 returns every slot up to the last tagged one)
  int32_t last = gk::kTraceCap;
  if (getenv("GK_TRACE_ALL")) {
    while (last > 1 && g->last_ctrl.tag[last - 1] == 0) last--;
  }
  int32_t k = 0;
  for (int32_t i = 0; i < last; i++) {
    if (i > 0 && g->last_ctrl.tag[i] == 0 && !getenv("GK_TRACE_ALL")) break;
    if (k < cap) {
      if (ts_ns) ts_ns[k] = g->last_ctrl.ts[i];
      if (tags) tags[k] = i == 0 ? 'S' : (char)g->last_ctrl.tag[i];
    }
    k++;
  }
  *count = k;
  return GK_OK;
}

gk_status gk_bfs_byte_model(gk_graph* g, const gk_step* steps, int32_t num_steps, double* b_sec,
                            double* b_use) {
  if (!g || !b_sec || !b_use || (num_steps > 0 && !steps)) return fail(GK_ERR_INVALID, "null argument");
  if (!g->depth || !g->depth_valid)
    return fail(GK_ERR_INVALID, "byte model needs the last gk_bfs to record depths");
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  std::vector<char> dirs(std::max(num_steps, 1));
  for (int i = 0; i < num_steps; i++) dirs[i] = (char)steps[i].dir;
  gk::BfsParams p{};
  p.n = g->n;
  p.out_off = g->out_off;
  p.out_nb = g->out_nb;
  p.in_off = g->in_off;
  p.in_nb = g->in_nb;
  CK(gk::byte_model(p, g->depth, dirs.data(), num_steps, nullptr, b_sec, b_use, g->stream), "byte model");
  return GK_OK;
}

gk_status gk_bfs_verify(gk_graph* g, uint32_t source, int64_t* errors) {
  if (!g || !errors) return fail(GK_ERR_INVALID, "null argument");
  if (!g->depth || !g->depth_valid)
    return fail(GK_ERR_INVALID, "verification needs the last gk_bfs to record depths");
  if ((int64_t)source >= g->n) return fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  long long e8[8];
  CK(gk::verify_bfs(g->out_off, g->out_nb, g->parent, g->depth, g->n, source, e8, g->stream), "verify");
  for (int i = 0; i < 8; i++) errors[i] = e8[i];
  return GK_OK;
}

// Brandes betweenness over the given sources (betweenness.hpp:84-145): one
// cooperative launch per source accumulates into device scores, then one
// max-normalisation.  Validation order and messages follow
// betweenness.hpp:86-93.  The whole call is one trial: its workspace
// (sigma/delta, successor bits, level data, traversal scratch) is taken from
// the pool inside the timed region and returned at its end.
gk_status gk_brandes(gk_graph* g, const uint32_t* sources, int64_t num_sources, float* scores_out,
                     double* device_ms) {
  NvtxRange nvtx_range("gk_brandes");
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  if (!sources || num_sources <= 0) return fail(GK_ERR_BAD_PARAM, "betweenness requires at least one source");
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  for (int64_t i = 0; i < num_sources; i++) {
    if ((int64_t)sources[i] >= g->n) return fail(GK_ERR_SOURCE_RANGE, "betweenness source out of range");
    int64_t o[2];
    CK(cudaMemcpy(o, g->out_off + sources[i], sizeof(o), cudaMemcpyDeviceToHost), "read degree");
    if (o[1] == o[0]) return fail(GK_ERR_BAD_PARAM, "betweenness source has zero out-degree");
  }
  const int64_t n = g->n;
  const int64_t w32 = (n + 31) / 32;
  g->last_valid = 0;  // the trace now describes Brandes
  g->depth_valid = 0;
  cudaStream_t s = g->stream;
  const size_t sz_sd = up(sizeof(double2) * std::max<int64_t>(n, 1)),
               sz_succ = up(sizeof(uint32_t) * ((g->m + 31) / 32 + 1)),
               sz_sc = up(sizeof(float) * std::max<int64_t>(n, 1) + 16), sz_dep = up(sizeof(int32_t) * (n + 4)),
               sz_bd = up(sizeof(int64_t) * (n + 2)), sz_lv = up(sizeof(uint32_t) * gk::kBcMaxPull * (w32 + 4)),
               sz_lvd = up(sizeof(long long) * gk::kBcMaxPull), sz_bits = 2 * bitmap_bytes(n),
               sz_q = up(sizeof(uint32_t) * (n + 1)), sz_ch = up(sizeof(gk::Chunk) * g->chunk_cap),
               sz_ctrl = up(sizeof(gk::Ctrl)), sz_st = up(sizeof(gk_step) * g->step_cap);
  const size_t total = sz_sd + sz_succ + sz_sc + sz_dep + sz_bd + sz_lv + sz_lvd + sz_bits + sz_q + sz_ch + sz_ctrl +
                       sz_st;
  CK(cudaEventRecord(g->ev0, s), "event record");
  char* w = nullptr;
  CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&w), total, g->pool, s), "allocate brandes workspace");
  gk::BfsParams p{};
  size_t at = 0;
  auto carve = [&](size_t sz) {
    char* r = w + at;
    at += sz;
    return r;
  };
  p.bc_sd = reinterpret_cast<double2*>(carve(sz_sd));
  p.bc_succ = reinterpret_cast<uint32_t*>(carve(sz_succ));
  p.bc_scores = reinterpret_cast<float*>(carve(sz_sc));
  p.depth = reinterpret_cast<int32_t*>(carve(sz_dep));
  p.bc_bounds = reinterpret_cast<int64_t*>(carve(sz_bd));
  p.bc_bounds_cap = n + 2;
  p.bc_lv = reinterpret_cast<uint32_t*>(carve(sz_lv));
  p.bc_lvw = w32 + 4;
  p.bc_lvdeg = reinterpret_cast<long long*>(carve(sz_lvd));
  p.visited = reinterpret_cast<uint32_t*>(carve(sz_bits));
  p.bm0 = p.visited + bitmap_bytes(n) / 4;
  p.queue = reinterpret_cast<uint32_t*>(carve(sz_q));
  p.chunks = reinterpret_cast<gk::Chunk*>(carve(sz_ch));
  p.ctrl = reinterpret_cast<gk::Ctrl*>(carve(sz_ctrl));
  p.steps = reinterpret_cast<gk_step*>(carve(sz_st));
  p.n = n;
  p.m = g->m;
  p.w32 = w32;
  p.out_off = g->out_off;
  p.out_nb = g->out_nb;
  p.in_off = g->in_off;
  p.in_nb = g->in_nb;
  p.chunk_cap = g->chunk_cap;
  p.step_cap = g->step_cap;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  if (const char* wd = getenv("GK_WATCHDOG_MS")) p.timeout_ns = strtoull(wd, nullptr, 10) * 1000000ull;
  p.stop_after = 0xffffffffu;
  p.dead = g->dead;
  p.live = g->live;
  set_compact_offsets(g, p);
  if (getenv("GK_BC_NO_PULL")) p.bc_lv = nullptr;  // top-down only (the reference's forward)
  gk_status st = GK_OK;
  cudaError_t e = cudaMemsetAsync(p.bc_scores, 0, sizeof(float) * n, s);
  for (int64_t i = 0; i < num_sources && !e && st == GK_OK; i++) {
    p.src = sources[i];
    if ((e = gk::bc_launch(p, g->device, s))) break;
    gk::Ctrl& ctrl = g->last_ctrl;  // kept for gk_bfs_trace (phase timings of the last source)
    if ((e = cudaMemcpyAsync(&ctrl, p.ctrl, sizeof(ctrl), cudaMemcpyDeviceToHost, s))) break;
    if ((e = cudaStreamSynchronize(s))) break;
    g->last_valid = 1;
    const int err = ctrl.error;
    if (err == 2) st = fail(GK_ERR_TIMEOUT, "brandes kernel watchdog fired (grid barrier timeout)");
    else if (err == 3) st = fail(GK_ERR_CUDA, "brandes kernel: chunk buffer overflow");
    else if (err == 4) st = fail(GK_ERR_CUDA, "brandes kernel: level bound buffer overflow");
    else if (err) st = fail(GK_ERR_CUDA, "brandes kernel failed");
  }
  if (!e && st == GK_OK) e = gk::bc_normalize(p.bc_scores, n, p.bc_scores + n, s);
  if (!e && st == GK_OK) e = cudaEventRecord(g->ev1, s);
  if (!e && st == GK_OK && scores_out)
    e = copy_out(g, scores_out, p.bc_scores, sizeof(float) * n, s);
  cudaFreeAsync(w, s);
  const cudaError_t es = cudaStreamSynchronize(s);
  if (!e) e = es;
  if (e) return cuda_fail(e, "brandes");
  if (st != GK_OK) return st;
  if (device_ms) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1), "event time");
    *device_ms = ms;
  }
  return GK_OK;
}

void* gk_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocDefault) != cudaSuccess) {
    g_last_error = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void gk_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
