// gk_shard.cu -- host side of the sharded traversal:
// one rank's rows and exchange buffers, their wiring to the other ranks,
// and the launches of bfs_sharded (gk_bfs_sharded.cu).
//
// Rank r of P owns vertices [r*block, min(n, (r+1)*block)), block =
// ceil(n/P) rounded up to 1024 (whole 32-word bottom-up tasks).  A rank
// holds the CSR rows of its vertices (global neighbour ids) and, for the
// traversal, full-n replicated bitmaps (visited, front/next, claims) in one
// allocation its peers map, plus the replicated dead bitmap (graph layout).
// Everything else a traversal touches -- owned parents and depths, queue,
// claim list, heavy chunks, control block, step log -- comes from the
// shard's pool inside the timed region; the mapped bitmaps are
// re-initialised by the kernel each trial.
//
// Wiring:
//   * ranks in one process on one device (gk_shard_join_local): one
//     cooperative launch runs every rank, cpr CTAs each -- the single-GPU
//     emulation of the multi-device run (B200_PROFILING.md: ranks that wait
//     on one another must not be separate launches on one GPU);
//   * one process per device (gk_shard_export / gk_shard_connect / a host
//     barrier / gk_shard_gather_dead): CUDA IPC handles of
//     every rank's bitmaps and of rank 0's cross-rank control block,
//     exchanged by the caller (torch.distributed in dist.py); every rank
//     then launches its own kernel and the ranks meet on the device.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gk_internal.cuh"

struct gk_shard {
  int device = 0;
  int rank = 0, nranks = 1;
  int64_t n = 0, lo = 0, hi = 0, nloc = 0, block = 0, m = 0;
  int64_t m_total = 0, live_total = 0;
  int64_t* off = nullptr;  // owned rows, local offsets (row i = vertex lo + i)
  uint32_t* off32 = nullptr;  // their compact form (m < 2^33), or null
  uint32_t off_hi = 0xffffffffu;  // global id of the carry vertex
  uint32_t* nb = nullptr;
  uint32_t* bm = nullptr;    // 4 full-n bitmaps (visited, front/next pair, claims), peer-mapped
  uint32_t* dead = nullptr;  // full-n dead bitmap (replicated graph layout)
  int32_t* parent = nullptr; // owned parents (peers store remote claims here), re-initialised per trial
  size_t wbytes = 0;         // bytes per full-n bitmap
  gk::XCtrl* x = nullptr;    // rank 0 of a multi-device group: cross-rank barrier + counters
  cudaMemPool_t pool = nullptr;
  cudaStream_t stream = nullptr;  // caller's stream (gk_shard_set_stream) or own
  cudaStream_t own_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  gk::BfsLaunch launch;
  bool connected = false;
  std::vector<gk_shard*> group;                  // local group: every rank's shard (this device)
  gk::ShardView peer[gk::kMaxRanks] = {};        // multi-device: peers' bitmaps (IPC-mapped)
  std::vector<void*> ipc_opened;
  gk::XCtrl* xpeer = nullptr;     // multi-device: rank 0's XCtrl as mapped here
  unsigned long long xsyncs = 0;  // cross-rank barriers passed by earlier traversals
  gk::Ctrl last_ctrl;
  long long launches = 0;
  unsigned long long* acc = nullptr;
};

namespace {

thread_local std::string g_shard_err;
gk_status shard_fail(gk_status st, const std::string& m) {
  g_shard_err = m;
  return st;
}
#define SCK(call, what)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return shard_fail(e_ == cudaErrorMemoryAllocation ? GK_ERR_OOM : GK_ERR_CUDA,            \
                        std::string(what) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

constexpr size_t kAlign = 256;
size_t up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

int64_t block_of(int64_t n, int nranks) {
  const int64_t b = (n + nranks - 1) / nranks;
  return (b + 1023) / 1024 * 1024;
}

void owned_range(int64_t n, int64_t block, int q, int64_t* lo, int64_t* hi) {
  *lo = std::min<int64_t>(n, q * block);
  *hi = std::min<int64_t>(n, *lo + block);
}

// Bitmap words a rank owns (none for an empty rank, lo = hi = n).
int64_t words_of(int64_t lo, int64_t hi) { return hi > lo ? (hi + 31) / 32 - lo / 32 : 0; }

// Bytes one traversal's exchanges bring into rank r: every step all-gathers
// next (the other ranks' owned words), every top-down step also reduces the
// claims over r's own words from every other rank.
int64_t bytes_in(const gk_shard* s, const gk_step* steps, int64_t k) {
  int64_t others = 0;
  for (int q = 0; q < s->nranks; q++) {
    if (q == s->rank) continue;
    int64_t lo, hi;
    owned_range(s->n, s->block, q, &lo, &hi);
    others += words_of(lo, hi) * 4;
  }
  const int64_t mine = words_of(s->lo, s->hi) * 4 * (s->nranks - 1);
  int64_t b = 0;
  for (int64_t i = 0; i < k; i++) b += others + (steps[i].dir == 'T' ? mine : 0);
  return b;
}

gk_status shard_setup(gk_shard* s) {
  const int64_t w32 = (s->n + 31) / 32;
  s->wbytes = up((size_t)w32 * 4 + 64);
  SCK(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking), "stream");
  s->stream = s->own_stream;
  SCK(cudaEventCreate(&s->ev0), "event");
  SCK(cudaEventCreate(&s->ev1), "event");
  SCK(cudaMalloc(&s->acc, sizeof(unsigned long long) * 4), "alloc acc");
  SCK(gk::shard_configure(s->device, &s->launch), "configure sharded kernel");
  SCK(cudaMalloc(&s->bm, 4 * s->wbytes), "alloc bitmaps");
  SCK(cudaMalloc(&s->dead, s->wbytes), "alloc dead bitmap");
  SCK(cudaMalloc(&s->parent, sizeof(int32_t) * (s->nloc + 16)), "alloc parents");
  SCK(cudaMemset(s->dead, 0xff, s->wbytes), "dead bitmap");  // the peers' words are gathered when wired
  // owned words from the owned rows (undirected: in-degree = out-degree)
  int64_t live = 0;
  SCK(gk::dead_bitmap(s->off, s->nloc, s->dead + s->lo / 32, &live, nullptr), "dead bitmap");
  // the rows' compact offsets, read by the sharded kernel's offset loads
  // like the single-device kernel's (gk_capi.cu setup_graph)
  if (s->m < (int64_t(2) << 32) && !getenv("GK_NO_OFF32")) {
    uint32_t* hi = nullptr;
    SCK(cudaMalloc(&s->off32, sizeof(uint32_t) * (size_t)(s->nloc + 1) + 64), "alloc compact offsets");
    SCK(cudaMalloc(&hi, sizeof(uint32_t)), "alloc compact offsets");
    SCK(cudaMemset(hi, 0xff, sizeof(uint32_t)), "compact offsets");
    SCK(gk::compact_offsets(s->off, s->nloc, s->off32, hi, (int)(s->m >> 32), nullptr), "compact offsets");
    uint32_t hl = 0xffffffffu;
    SCK(cudaMemcpy(&hl, hi, sizeof(hl), cudaMemcpyDeviceToHost), "compact offsets");
    cudaFree(hi);
    s->off_hi = hl == 0xffffffffu ? 0xffffffffu : (uint32_t)(s->lo + hl);
  }
  if (s->rank == 0) {
    SCK(cudaMalloc(&s->x, sizeof(gk::XCtrl)), "alloc cross-rank control");
    SCK(cudaMemset(s->x, 0, sizeof(gk::XCtrl)), "cross-rank control");
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = s->device;
  SCK(cudaMemPoolCreate(&s->pool, &props), "memory pool");
  uint64_t keep = UINT64_MAX;
  SCK(cudaMemPoolSetAttribute(s->pool, cudaMemPoolAttrReleaseThreshold, &keep), "memory pool");
  SCK(cudaDeviceSynchronize(), "shard setup");
  return GK_OK;
}

void shard_free(gk_shard* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : {(void*)s->off, (void*)s->off32, (void*)s->nb, (void*)s->bm, (void*)s->dead, (void*)s->parent,
                  (void*)s->x, (void*)s->acc}) cudaFree(p);
  if (s->pool) cudaMemPoolDestroy(s->pool);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
}

gk_status shard_new(int64_t n, int rank, int nranks, int device, gk_shard** out) {
  if (!out || nranks < 1 || nranks > gk::kMaxRanks || rank < 0 || rank >= nranks || n < 1 ||
      n > (int64_t(1) << 31))
    return shard_fail(GK_ERR_INVALID, "bad shard spec (1 <= ranks <= 8, 0 <= rank < ranks, 1 <= n <= 2^31)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return shard_fail(GK_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
  if (device < 0 || device >= ndev) return shard_fail(GK_ERR_INVALID, "device index out of range");
  SCK(cudaSetDevice(device), "cudaSetDevice");
  auto* s = new gk_shard;
  s->device = device;
  s->rank = rank;
  s->nranks = nranks;
  s->n = n;
  s->block = block_of(n, nranks);
  owned_range(n, s->block, rank, &s->lo, &s->hi);
  s->nloc = s->hi - s->lo;
  *out = s;
  return GK_OK;
}

// Owned-range hub expansion (gk_internal.cuh OwnEnt) for a rank run by
// `ctas` CTAs: each takes a range of all n target ids, its slice of the
// claims bitmap in shared memory; off when the slice does not fit.
struct OwnGeom {
  int ranges = 0, win_log = 0;
  int64_t span_w = 0, cap = 0, dmin = 32768;
  size_t stage_bytes = 0;
};
OwnGeom own_geometry(const gk_shard* s, int ctas) {
  OwnGeom g;
  const int64_t w32 = (s->n + 31) / 32;
  const int64_t span_w = ((w32 + ctas - 1) / ctas + 3) & ~int64_t(3);
  if (getenv("GK_NO_OWN") || (size_t)span_w * 4 > s->launch.smem_keep_occ) return g;
  if (const char* dm = getenv("GK_OWN_DMIN")) g.dmin = std::max<int64_t>(1, strtoll(dm, nullptr, 10));
  int wl = 0;
  while ((int64_t(2) << wl) <= span_w) wl++;
  const int64_t nwin = (32 * span_w + (int64_t(1) << wl) - 1) >> wl;
  g.ranges = ctas;
  g.win_log = wl;
  g.span_w = span_w;
  g.cap = s->m / g.dmin + 1;
  g.stage_bytes = sizeof(uint2) * (size_t)ctas * (size_t)(nwin << wl);
  return g;
}

struct ShardTrial {
  void* block = nullptr;
  int32_t* depth = nullptr;  // owned range
  uint32_t* queue = nullptr;
  gk::OwnEnt* own_list = nullptr;
  uint2* own_stage = nullptr;
  OwnGeom own;
  gk::Chunk* chunks = nullptr;
  gk::Ctrl* ctrl = nullptr;
  gk_step* steps = nullptr;
  int64_t chunk_cap = 0, step_cap = 0;
};

// One pool block per traversal: owned depths (parity runs), the queue of
// owned frontier windows and long lists, heavy chunks, the control block and
// the step log.  (Owned parents live in the mapped s->parent.)
cudaError_t trial_alloc(gk_shard* s, ShardTrial* t, bool depth, int ctas, cudaStream_t st) {
  const int64_t nl = std::max<int64_t>(s->nloc, 1);
  t->own = own_geometry(s, ctas);
  const size_t sz_ol = t->own.ranges ? up(sizeof(gk::OwnEnt) * t->own.cap) : 0,
               sz_os = t->own.ranges ? up(t->own.stage_bytes) : 0;
  t->chunk_cap = 2 * (s->m / 1024) + 65536;
  t->step_cap = std::min<int64_t>(s->n + 2, int64_t(1) << 20);
  const size_t sz_d = depth ? up(4 * nl) : 0, sz_q = up(4 * (2 * nl + 64)),
               sz_c = up(sizeof(gk::Chunk) * t->chunk_cap), sz_ctrl = up(sizeof(gk::Ctrl)),
               sz_s = up(sizeof(gk_step) * t->step_cap);
  cudaError_t e = cudaMallocFromPoolAsync(&t->block, sz_d + sz_q + sz_c + sz_ctrl + sz_s + sz_ol + sz_os, s->pool, st);
  if (e) return e;
  char* b = static_cast<char*>(t->block);
  if (t->own.ranges) {
    t->own_list = reinterpret_cast<gk::OwnEnt*>(b);
    t->own_stage = reinterpret_cast<uint2*>(b + sz_ol);
    b += sz_ol + sz_os;
  }
  t->depth = depth ? reinterpret_cast<int32_t*>(b) : nullptr;
  b += sz_d;
  t->queue = reinterpret_cast<uint32_t*>(b);
  b += sz_q;
  t->chunks = reinterpret_cast<gk::Chunk*>(b);
  b += sz_c;
  t->ctrl = reinterpret_cast<gk::Ctrl*>(b);
  b += sz_ctrl;
  t->steps = reinterpret_cast<gk_step*>(b);
  return cudaSuccess;
}

gk::ShardView view_of(const gk_shard* s, const ShardTrial& t) {
  gk::ShardView v{};
  v.off = s->off - s->lo;  // shifted: off[v] for owned v
  v.off32 = s->off32 ? s->off32 - s->lo : nullptr;
  v.off_hi = s->off_hi;
  v.nb = s->nb;
  v.parent = s->parent - s->lo;
  v.depth = t.depth ? t.depth - s->lo : nullptr;
  v.queue = t.queue;
  v.own_list = t.own_list;
  v.own_stage = t.own_stage;
  v.own_cap = t.own.cap;
  v.chunks = t.chunks;
  v.chunk_cap = t.chunk_cap;
  for (int k = 0; k < 4; k++) v.bm[k] = s->bm + k * (s->wbytes / 4);
  v.dead = s->dead;
  v.lo = s->lo;
  v.hi = s->hi;
  return v;
}

gk::BfsParams base_params(const gk_shard* s, const ShardTrial& t, uint32_t source, int64_t alpha, int64_t beta,
                          int32_t strategy, int want_depth) {
  gk::BfsParams p{};
  p.n = s->n;
  p.m = s->m_total;
  p.w32 = (s->n + 31) / 32;
  p.src = source;
  p.strategy = strategy;
  p.alpha = alpha;
  p.beta = beta;
  p.want_depth = want_depth;
  p.live = s->live_total;
  p.ctrl = t.ctrl;
  p.steps = t.steps;
  p.step_cap = t.step_cap;
  p.bu_tw_log_max = 5;
  p.td_passes = 1;
  p.td_span = ((s->n + 31) / 32) * 32;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  if (const char* w = getenv("GK_WATCHDOG_MS")) p.timeout_ns = strtoull(w, nullptr, 10) * 1000000ull;
  p.stop_after = 0xffffffffu;
  if (t.own.ranges) {
    p.own_list = t.own_list;
    p.own_cap = t.own.cap;
    p.own_stage = t.own_stage;
    p.own_r = t.own.ranges;
    p.own_span_w = (int32_t)t.own.span_w;
    p.own_win_log = t.own.win_log;
    p.own_dmin = t.own.dmin;
  }
  return p;
}

gk_status check_source(const gk_shard* s, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy) {
  if ((int64_t)source >= s->n) return shard_fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  if (alpha <= 0 || beta <= 0) return shard_fail(GK_ERR_BAD_PARAM, "bfs alpha and beta must be positive");
  if (strategy < 0 || strategy > 2) return shard_fail(GK_ERR_BAD_PARAM, "unknown bfs strategy");
  if (!s->connected) return shard_fail(GK_ERR_INVALID, "shard not wired (gk_shard_join_local / gk_shard_connect)");
  return GK_OK;
}

gk_status kernel_status(const gk::Ctrl& c) {
  if (c.error == 2) return shard_fail(GK_ERR_TIMEOUT, "sharded bfs: barrier watchdog fired");
  if (c.error) return shard_fail(GK_ERR_CUDA, "sharded bfs: scratch buffer overflow");
  return GK_OK;
}

int64_t live_of(const uint32_t* dead_dev, int64_t n, gk_status* st) {
  std::vector<uint32_t> h((n + 31) / 32);
  if (cudaMemcpy(h.data(), dead_dev, 4 * h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
    *st = shard_fail(GK_ERR_CUDA, "dead bitmap D2H");
    return 0;
  }
  int64_t l = 0;
  for (uint32_t w : h) l += __builtin_popcount(~w);
  *st = GK_OK;
  return l;
}

}  // namespace

extern "C" {

GK_API const char* gk_shard_last_error(void) { return g_shard_err.c_str(); }

GK_API gk_status gk_shard_generate(int kind, int scale, int degree, uint64_t seed, int permute, int rank,
                                   int nranks, int device, gk_shard** out) {
  if (kind != 0 && kind != 1) return shard_fail(GK_ERR_INVALID, "generator kind must be 0 or 1");
  if (scale < 5 || scale > 31) return shard_fail(GK_ERR_INVALID, "sharded generator scale must be in [5, 31]");
  gk_shard* s = nullptr;
  gk_status st = shard_new(int64_t{1} << scale, rank, nranks, device, &s);
  if (st != GK_OK) return st;
  gk::DevCsr csr;
  std::string err;
  cudaError_t e = gk::build_generated(kind, scale, degree, seed, permute, s->lo, s->hi, &csr, &err);
  if (e != cudaSuccess) {
    shard_free(s);
    return shard_fail(GK_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  }
  s->off = csr.off;
  s->nb = csr.nb;
  s->m = csr.m;
  if ((st = shard_setup(s)) != GK_OK) {
    shard_free(s);
    return st;
  }
  *out = s;
  return GK_OK;
}

GK_API gk_status gk_shard_upload(int64_t n, int rank, int nranks, const int64_t* local_offsets,
                                 const uint32_t* neighbors, int device, gk_shard** out) {
  if (!local_offsets) return shard_fail(GK_ERR_INVALID, "null offsets");
  gk_shard* s = nullptr;
  gk_status st = shard_new(n, rank, nranks, device, &s);
  if (st != GK_OK) return st;
  s->m = local_offsets[s->nloc];
  cudaError_t e;
  if ((e = cudaMalloc(&s->off, sizeof(int64_t) * (s->nloc + 3))) ||
      (e = cudaMalloc(&s->nb, sizeof(uint32_t) * std::max<int64_t>(s->m, 1) + gk::kNbPad)) ||
      (e = cudaMemcpy(s->off, local_offsets, sizeof(int64_t) * (s->nloc + 1), cudaMemcpyHostToDevice)) ||
      (s->m && (e = cudaMemcpy(s->nb, neighbors, sizeof(uint32_t) * s->m, cudaMemcpyHostToDevice)))) {
    shard_free(s);
    return shard_fail(GK_ERR_CUDA, cudaGetErrorString(e));
  }
  bool off_ok = true, ids_ok = true;
  if ((e = gk::validate_csr(s->off, s->nb, s->nloc, s->m, s->n, &off_ok, &ids_ok, nullptr, nullptr)) || !off_ok ||
      !ids_ok) {
    shard_free(s);
    return shard_fail(GK_ERR_INVALID, e ? cudaGetErrorString(e) : "invalid shard rows");
  }
  if ((st = shard_setup(s)) != GK_OK) {
    shard_free(s);
    return st;
  }
  *out = s;
  return GK_OK;
}

GK_API void gk_shard_free(gk_shard* s) { shard_free(s); }

GK_API gk_status gk_shard_info(const gk_shard* s, int64_t* n, int64_t* lo, int64_t* hi, int64_t* arcs,
                               int64_t* block) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  if (n) *n = s->n;
  if (lo) *lo = s->lo;
  if (hi) *hi = s->hi;
  if (arcs) *arcs = s->m;
  if (block) *block = s->block;
  return GK_OK;
}

GK_API int64_t gk_shard_launches(const gk_shard* s) { return s ? s->launches : 0; }

GK_API gk_status gk_shard_download(const gk_shard* s, int64_t* local_offsets, uint32_t* neighbors) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  if (local_offsets) SCK(cudaMemcpy(local_offsets, s->off, 8 * (s->nloc + 1), cudaMemcpyDeviceToHost), "download");
  if (neighbors && s->m) SCK(cudaMemcpy(neighbors, s->nb, 4 * s->m, cudaMemcpyDeviceToHost), "download");
  return GK_OK;
}

GK_API gk_status gk_shard_set_stream(gk_shard* s, void* stream) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  s->stream = stream ? (cudaStream_t)stream : s->own_stream;
  return GK_OK;
}

GK_API gk_status gk_shard_join_local(gk_shard* const* shards, int nranks) {
  if (!shards || nranks < 1 || nranks > gk::kMaxRanks) return shard_fail(GK_ERR_INVALID, "bad group");
  for (int q = 0; q < nranks; q++)
    if (!shards[q] || shards[q]->rank != q || shards[q]->nranks != nranks || shards[q]->n != shards[0]->n ||
        shards[q]->device != shards[0]->device)
      return shard_fail(GK_ERR_INVALID, "group must be ranks 0..P-1 of one graph on one device");
  SCK(cudaSetDevice(shards[0]->device), "cudaSetDevice");
  int64_t m_total = 0;
  for (int q = 0; q < nranks; q++) m_total += shards[q]->m;
  for (int q = 0; q < nranks; q++)
    for (int p = 0; p < nranks; p++) {
      if (p == q) continue;
      const gk_shard* o = shards[p];
      const int64_t w0 = o->lo / 32, w1 = w0 + words_of(o->lo, o->hi);
      if (w1 > w0)
        SCK(cudaMemcpy(shards[q]->dead + w0, o->dead + w0, 4 * (w1 - w0), cudaMemcpyDeviceToDevice), "dead gather");
    }
  gk_status st;
  const int64_t live = live_of(shards[0]->dead, shards[0]->n, &st);
  if (st != GK_OK) return st;
  for (int q = 0; q < nranks; q++) {
    shards[q]->group.assign(shards, shards + nranks);
    shards[q]->m_total = m_total;
    shards[q]->live_total = live;
    shards[q]->connected = true;
  }
  return GK_OK;
}

GK_API int64_t gk_shard_handle_size(void) { return 3 * (int64_t)sizeof(cudaIpcMemHandle_t) + 64; }

GK_API gk_status gk_shard_export(const gk_shard* s, void* handle_out) {
  if (!s || !handle_out) return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  char* o = static_cast<char*>(handle_out);
  std::memset(o, 0, gk_shard_handle_size());
  cudaIpcMemHandle_t hb, hx, hp;
  SCK(cudaIpcGetMemHandle(&hb, s->bm), "ipc handle (bitmaps)");
  std::memcpy(o, &hb, sizeof(hb));
  if (s->rank == 0) {
    SCK(cudaIpcGetMemHandle(&hx, s->x), "ipc handle (control)");
    std::memcpy(o + sizeof(hb), &hx, sizeof(hx));
  }
  SCK(cudaIpcGetMemHandle(&hp, s->parent), "ipc handle (parents)");
  std::memcpy(o + 2 * sizeof(hb), &hp, sizeof(hp));
  const int64_t meta[4] = {s->rank, s->m, (int64_t)s->wbytes, s->nranks};
  std::memcpy(o + 3 * sizeof(cudaIpcMemHandle_t), meta, sizeof(meta));
  // the dead bitmap's owned words travel in the visited slot until gk_shard_gather_dead
  const int64_t w0 = s->lo / 32, w1 = w0 + words_of(s->lo, s->hi);
  if (w1 > w0) SCK(cudaMemcpy(s->bm + w0, s->dead + w0, 4 * (w1 - w0), cudaMemcpyDeviceToDevice), "publish dead");
  return GK_OK;
}

GK_API gk_status gk_shard_connect(gk_shard* s, const void* handles) {
  if (!s || !handles) return shard_fail(GK_ERR_INVALID, "null argument");
  if (!s->group.empty()) return shard_fail(GK_ERR_INVALID, "shard belongs to a local group");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  const char* h = static_cast<const char*>(handles);
  const int64_t hs = gk_shard_handle_size();
  int64_t m_total = 0;
  for (int q = 0; q < s->nranks; q++) {
    int64_t meta[4];
    std::memcpy(meta, h + q * hs + 3 * sizeof(cudaIpcMemHandle_t), sizeof(meta));
    if (meta[0] != q || meta[3] != s->nranks || meta[2] != (int64_t)s->wbytes)
      return shard_fail(GK_ERR_INVALID, "handles of a different group");
    m_total += meta[1];
    uint32_t* bm = s->bm;
    int32_t* par = s->parent;
    if (q != s->rank) {
      cudaIpcMemHandle_t hb, hp;
      std::memcpy(&hb, h + q * hs, sizeof(hb));
      std::memcpy(&hp, h + q * hs + 2 * sizeof(hb), sizeof(hp));
      void* p = nullptr;
      SCK(cudaIpcOpenMemHandle(&p, hb, cudaIpcMemLazyEnablePeerAccess), "map peer bitmaps");
      s->ipc_opened.push_back(p);
      bm = static_cast<uint32_t*>(p);
      SCK(cudaIpcOpenMemHandle(&p, hp, cudaIpcMemLazyEnablePeerAccess), "map peer parents");
      s->ipc_opened.push_back(p);
      par = static_cast<int32_t*>(p);
    }
    for (int k = 0; k < 4; k++) s->peer[q].bm[k] = bm + k * (s->wbytes / 4);
    int64_t lo, hi;
    owned_range(s->n, s->block, q, &lo, &hi);
    s->peer[q].parent = par - lo;
    s->peer[q].lo = lo;
    s->peer[q].hi = hi;
  }
  if (s->rank == 0) {
    s->xpeer = s->x;
  } else {
    cudaIpcMemHandle_t hx;
    std::memcpy(&hx, h + sizeof(cudaIpcMemHandle_t), sizeof(hx));
    void* p = nullptr;
    SCK(cudaIpcOpenMemHandle(&p, hx, cudaIpcMemLazyEnablePeerAccess), "map cross-rank control");
    s->ipc_opened.push_back(p);
    s->xpeer = static_cast<gk::XCtrl*>(p);
  }
  s->m_total = m_total;
  return GK_OK;
}

GK_API gk_status gk_shard_gather_dead(gk_shard* s) {
  if (!s || !s->group.empty() || !s->xpeer) return shard_fail(GK_ERR_INVALID, "call after gk_shard_connect");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  for (int q = 0; q < s->nranks; q++) {
    if (q == s->rank) continue;
    int64_t lo, hi;
    owned_range(s->n, s->block, q, &lo, &hi);
    const int64_t w0 = lo / 32, w1 = w0 + words_of(lo, hi);
    if (w1 > w0) SCK(cudaMemcpy(s->dead + w0, s->peer[q].bm[0] + w0, 4 * (w1 - w0), cudaMemcpyDefault), "gather dead");
  }
  gk_status st;
  s->live_total = live_of(s->dead, s->n, &st);
  if (st != GK_OK) return st;
  s->connected = true;
  return GK_OK;
}

GK_API gk_status gk_shard_group_bfs(gk_shard* s0, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy,
                                    int32_t* const* parents_out, int32_t* const* depths_out, gk_bfs_stats* stats) {
  if (!s0) return shard_fail(GK_ERR_INVALID, "null shard");
  gk_status st = check_source(s0, source, alpha, beta, strategy);
  if (st != GK_OK) return st;
  if (s0->group.empty() || s0->group[0] != s0) return shard_fail(GK_ERR_INVALID, "call on rank 0 of a local group");
  const int P = (int)s0->group.size();
  SCK(cudaSetDevice(s0->device), "cudaSetDevice");
  cudaStream_t str = s0->stream;
  const int want_depth = depths_out != nullptr;
  std::vector<ShardTrial> tr(P);
  SCK(cudaEventRecord(s0->ev0, str), "event");
  const int cpr = s0->launch.grid / P;
  for (int q = 0; q < P; q++) SCK(trial_alloc(s0->group[q], &tr[q], want_depth, cpr, str), "trial scratch");
  gk::ShardTab tab{};
  tab.nranks = P;
  tab.emulated = 1;
  tab.m_total = s0->m_total;
  tab.live_total = s0->live_total;
  tab.block = s0->block;
  for (int q = 0; q < P; q++) tab.v[q] = view_of(s0->group[q], tr[q]);
  gk::BfsParams p = base_params(s0, tr[0], source, alpha, beta, strategy, want_depth);
  p.cpr = cpr;
  SCK(gk::shard_launch(p, tab, cpr * P, str), "launch sharded bfs");
  SCK(cudaEventRecord(s0->ev1, str), "event");
  s0->launches++;
  SCK(cudaMemcpyAsync(&s0->last_ctrl, tr[0].ctrl, sizeof(gk::Ctrl), cudaMemcpyDeviceToHost, str), "read ctrl");
  SCK(cudaStreamSynchronize(str), "sharded bfs");
  st = kernel_status(s0->last_ctrl);
  int64_t reached = 0, edges = 0;
  for (int q = 0; q < P && st == GK_OK; q++) {
    gk_shard* s = s0->group[q];
    if (parents_out && parents_out[q] && s->nloc)
      SCK(cudaMemcpyAsync(parents_out[q], s->parent, 4 * s->nloc, cudaMemcpyDeviceToHost, str), "D2H parent");
    if (depths_out && depths_out[q] && s->nloc)
      SCK(cudaMemcpyAsync(depths_out[q], tr[q].depth, 4 * s->nloc, cudaMemcpyDeviceToHost, str), "D2H depth");
    if (stats && stats->want_counts) {
      unsigned long long two[2];
      SCK(gk::count_reached(s->parent, s->off, s->nloc, s0->acc, str), "count reached");
      SCK(cudaMemcpyAsync(two, s0->acc, sizeof(two), cudaMemcpyDeviceToHost, str), "read counts");
      SCK(cudaStreamSynchronize(str), "count reached");
      reached += (int64_t)two[0];
      edges += (int64_t)two[1];
    }
  }
  if (st == GK_OK && stats) {
    float ms = 0;
    SCK(cudaEventElapsedTime(&ms, s0->ev0, s0->ev1), "event time");
    stats->device_ms = ms;
    stats->num_steps = (int32_t)s0->last_ctrl.num_steps;
    stats->reached = reached;
    stats->component_edges = edges / 2;
    if (stats->steps && stats->max_steps > 0) {
      const int64_t k = std::min<int64_t>({(int64_t)stats->max_steps, s0->last_ctrl.num_steps, tr[0].step_cap});
      if (k > 0)
        SCK(cudaMemcpyAsync(stats->steps, tr[0].steps, sizeof(gk_step) * k, cudaMemcpyDeviceToHost, str), "steps");
    }
  }
  for (int q = 0; q < P; q++) cudaFreeAsync(tr[q].block, str);
  SCK(cudaStreamSynchronize(str), "sharded bfs");
  return st;
}

GK_API gk_status gk_shard_bfs(gk_shard* s, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy,
                              int32_t* parent_out, int32_t* depth_out, gk_bfs_stats* stats, int64_t* bytes_in_out) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  gk_status st = check_source(s, source, alpha, beta, strategy);
  if (st != GK_OK) return st;
  if (!s->group.empty()) return shard_fail(GK_ERR_INVALID, "local group: use gk_shard_group_bfs");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  cudaStream_t str = s->stream;
  const int want_depth = depth_out != nullptr;
  ShardTrial tr;
  SCK(cudaEventRecord(s->ev0, str), "event");
  SCK(trial_alloc(s, &tr, want_depth, s->launch.grid, str), "trial scratch");
  gk::ShardTab tab{};
  tab.nranks = s->nranks;
  tab.emulated = 0;
  tab.rank = s->rank;
  tab.m_total = s->m_total;
  tab.live_total = s->live_total;
  tab.block = s->block;
  for (int q = 0; q < s->nranks; q++) tab.v[q] = s->peer[q];
  tab.v[s->rank] = view_of(s, tr);
  tab.x = s->xpeer;
  tab.xbase = s->xsyncs;
  tab.force_x = getenv("GK_SHARD_FORCE_X") ? 1 : 0;  // tests: the cross-device protocol with one rank
  gk::BfsParams p = base_params(s, tr, source, alpha, beta, strategy, want_depth);
  SCK(gk::shard_launch(p, tab, s->launch.grid, str), "launch sharded bfs");
  SCK(cudaEventRecord(s->ev1, str), "event");
  s->launches++;
  SCK(cudaMemcpyAsync(&s->last_ctrl, tr.ctrl, sizeof(gk::Ctrl), cudaMemcpyDeviceToHost, str), "read ctrl");
  SCK(cudaStreamSynchronize(str), "sharded bfs");
  s->xsyncs += s->last_ctrl.xsyncs;
  st = kernel_status(s->last_ctrl);
  if (st == GK_OK) {
    const int64_t k = std::min<int64_t>(s->last_ctrl.num_steps, tr.step_cap);
    std::vector<gk_step> steps(std::max<int64_t>(k, 1));
    if (k > 0) SCK(cudaMemcpyAsync(steps.data(), tr.steps, sizeof(gk_step) * k, cudaMemcpyDeviceToHost, str), "steps");
    if (parent_out && s->nloc)
      SCK(cudaMemcpyAsync(parent_out, s->parent, 4 * s->nloc, cudaMemcpyDeviceToHost, str), "D2H parent");
    if (depth_out && s->nloc)
      SCK(cudaMemcpyAsync(depth_out, tr.depth, 4 * s->nloc, cudaMemcpyDeviceToHost, str), "D2H depth");
    unsigned long long two[2] = {0, 0};
    if (stats && stats->want_counts) {
      SCK(gk::count_reached(s->parent, s->off, s->nloc, s->acc, str), "count reached");
      SCK(cudaMemcpyAsync(two, s->acc, sizeof(two), cudaMemcpyDeviceToHost, str), "read counts");
    }
    SCK(cudaStreamSynchronize(str), "D2H");
    if (bytes_in_out) *bytes_in_out = bytes_in(s, steps.data(), k);
    if (stats) {
      float ms = 0;
      SCK(cudaEventElapsedTime(&ms, s->ev0, s->ev1), "event time");
      stats->device_ms = ms;
      stats->num_steps = (int32_t)s->last_ctrl.num_steps;
      stats->reached = (int64_t)two[0];
      stats->component_edges = (int64_t)two[1];  // out-arcs of owned reached vertices (sum over ranks / 2)
      if (stats->steps && stats->max_steps > 0)
        std::memcpy(stats->steps, steps.data(), sizeof(gk_step) * std::min<int64_t>(stats->max_steps, k));
    }
  }
  cudaFreeAsync(tr.block, str);
  SCK(cudaStreamSynchronize(str), "sharded bfs");
  return st;
}

GK_API gk_status gk_shard_trace(const gk_shard* s, uint64_t* ts_ns, char* tags, int32_t cap, int32_t* count) {
  if (!s || !count) return shard_fail(GK_ERR_INVALID, "null argument");
  int32_t k = 0;
  for (int32_t i = 0; i < gk::kTraceCap; i++) {
    if (i > 0 && s->last_ctrl.tag[i] == 0) break;
    if (k < cap) {
      if (ts_ns) ts_ns[k] = s->last_ctrl.ts[i];
      if (tags) tags[k] = i == 0 ? 'S' : (char)s->last_ctrl.tag[i];
    }
    k++;
  }
  *count = k;
  return GK_OK;
}

GK_API gk_status gk_shard_bytes_in(const gk_shard* s, int32_t rank, const gk_step* steps, int32_t num_steps,
                                   int64_t* out) {
  if (!s || !out || rank < 0 || rank >= s->nranks || (num_steps > 0 && !steps))
    return shard_fail(GK_ERR_INVALID, "bad argument");
  const gk_shard* r = s->group.empty() ? s : s->group[rank];
  if (r->rank != rank) return shard_fail(GK_ERR_INVALID, "rank not held here");
  *out = bytes_in(r, steps, num_steps);
  return GK_OK;
}

}  // extern "C"
