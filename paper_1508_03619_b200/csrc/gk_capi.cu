// gk_capi.cu -- the C ABI of include/gk_bfs.h.
//
// Every entry point catches failures and returns a gk_status with a
// thread-local message; nothing throws across the boundary.  There is no
// CPU path: without a device, compute entry points fail with
// GK_ERR_NO_DEVICE.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gk_internal.cuh"

namespace {

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
  if (g->in_off && g->in_off != g->out_off) cudaFree(g->in_off);
  if (g->in_nb && g->in_nb != g->out_nb) cudaFree(g->in_nb);
  cudaFree(g->out_off);
  cudaFree(g->out_nb);
  cudaFree(g->parent);
  cudaFree(g->parent2);
  cudaFree(g->depth);
  cudaFree(g->bits);
  cudaFree(g->head);
  cudaFree(g->head2);
  cudaFree(g->bc_sd);
  cudaFree(g->bc_succ);
  cudaFree(g->bc_scores);
  cudaFree(g->bc_bounds);
  cudaFree(g->bc_lv);
  cudaFree(g->bc_lvdeg);
  cudaFree(g->hbase);
  cudaFree(g->deg16);
  cudaFree(g->hv_bits);
  cudaFree(g->hv_base);
  cudaFree(g->own_split);
  cudaFree(g->own_list);
  cudaFree(g->own_stage);
  cudaFree(g->queue);
  cudaFree(g->chunks);
  cudaFree(g->ctrl);
  cudaFree(g->steps);
  cudaFree(g->acc);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->stream) cudaStreamDestroy(g->stream);
  if (g->cstream) cudaStreamDestroy(g->cstream);
  delete g;
}

// Workspace sized for n vertices / m arcs; reused across trials and
// re-initialised inside the timed kernel.
gk_status alloc_workspace(gk_graph* g) {
  const int64_t n = g->n;
  const int64_t w32 = (n + 31) / 32;
  const size_t wbytes = ((size_t)w32 * 4 + 15) & ~size_t(15);
  CK(cudaMalloc(&g->parent, sizeof(int32_t) * std::max<int64_t>(n, 4) + 16), "alloc parent");
  // visited | front | next bitmaps in one block so one L2 access-policy
  // window can keep them resident while the graph streams past.
  CK(cudaMalloc(&g->bits, 4 * wbytes + 64), "alloc bitmaps");
  g->visited = g->bits;
  g->bm0 = g->bits + wbytes / 4;
  g->bm1 = g->bits + 2 * (wbytes / 4);
  g->dead = g->bits + 3 * (wbytes / 4);
  CK(cudaMalloc(&g->queue, sizeof(uint32_t) * (n + 1)), "alloc queue");
  g->chunk_cap = 2 * (g->m / 1024) + 65536;  // >= 4 x warps when chunks shrink to 128 edges
  CK(cudaMalloc(&g->chunks, sizeof(gk::Chunk) * g->chunk_cap), "alloc chunks");
  CK(cudaMalloc(&g->ctrl, 2 * sizeof(gk::Ctrl)), "alloc ctrl");
  CK(cudaMemset(g->ctrl, 0, 2 * sizeof(gk::Ctrl)), "clear ctrl");
  g->step_cap = std::min<int64_t>(n + 2, int64_t(1) << 20);
  CK(cudaMalloc(&g->steps, sizeof(gk_step) * g->step_cap), "alloc step log");
  CK(cudaMalloc(&g->acc, sizeof(unsigned long long) * 8), "alloc acc");
  CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking), "stream");
  CK(cudaEventCreate(&g->ev0), "event");
  CK(cudaEventCreate(&g->ev1), "event");
  CK(gk::bfs_configure(g->device, &g->launch), "configure bfs kernel");
  if (getenv("GK_NO_FRONT_SMEM")) g->launch.smem_front_max = 0;  // tests: large-graph paths on small graphs
  CK(gk::dead_bitmap(g->in_off, n, g->dead, g->stream), "dead-vertex bitmap");
  CK(cudaMalloc(&g->hbase, sizeof(uint32_t) * std::max<int64_t>(w32, 1)), "alloc head index");
  CK(gk::build_head(g->in_off, g->in_nb, n, g->dead, g->hbase, &g->head, &g->head2, &g->live, g->stream), "in-list heads");
  CK(cudaMalloc(&g->deg16, std::max<int64_t>(w32, 1) * 64), "alloc degree array");
  CK(gk::build_deg16(g->out_off, n, g->deg16, g->stream), "degree array");
  // Owned-range hub expansion (gk_internal.cuh OwnEnt): one target range per
  // CTA of the launch, its slice of the next bitmap in dynamic shared memory
  // without lowering the occupancy; hubs (out-degree >= 8192; 4096 and 16384
  // measured within 0.4% on kron27) get split rows.
  // Off when the slice does not fit (n > ~2^27 at 296 CTAs) or memory is short.
  {
    const int r = g->launch.grid;
    const int64_t span_w = ((w32 + r - 1) / r + 3) & ~int64_t(3);
    const bool fits = (size_t)span_w * 4 <= g->launch.smem_keep_occ && (size_t)w32 * 4 > g->launch.smem_front_max;
    if (fits && !getenv("GK_NO_OWN")) {
      int64_t nh = 0;
      const char* dm = getenv("GK_OWN_DMIN");  // tests: hubs on small graphs
      const int64_t dmin = dm ? std::max<int64_t>(1, strtoll(dm, nullptr, 10)) : 8192;
      CK(gk::build_own(g->out_off, g->out_nb, n, dmin, r, span_w, size_t(1) << 30, &g->hv_bits, &g->hv_base,
                       &g->own_split, &nh, g->stream),
         "owned-range split rows");
      if (nh > 0) {
        CK(cudaMalloc(&g->own_list, sizeof(gk::OwnEnt) * nh), "alloc owned-range list");
        int wl = 0;
        while ((int64_t(2) << wl) <= span_w) wl++;
        const int64_t nwin = (32 * span_w + (int64_t(1) << wl) - 1) >> wl;  // <= kOwnWin
        CK(cudaMalloc(&g->own_stage, sizeof(uint2) * (size_t)r * (size_t)(nwin << wl)), "alloc owned-range log");
        g->own_win_log = wl;
        g->own_r = r;
        g->own_span_w = span_w;
        g->own_dmin = dmin;
      }
    }
  }
  CK(cudaStreamSynchronize(g->stream), "dead-vertex bitmap");
  // L2 persisting window over the bitmaps: off by default since the
  // pending-list / sparse / pushed-step kernels (kron27 +2.6 %, urand27
  // +1.4 % without it; a 1-bitmap window measured the same as none); the
  // bitmap loads keep their evict_last hints.  GK_L2_PERSIST=1 restores it.
  const char* pers = getenv("GK_L2_PERSIST");
  if (pers && atoi(pers) != 0) {
    int max_win = 0, max_pers = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, g->device);
    cudaDeviceGetAttribute(&max_pers, cudaDevAttrMaxPersistingL2CacheSize, g->device);
    const char* nbm = getenv("GK_L2_BITMAPS");  // A-B: bitmaps in the window (visited, bm0, bm1, dead)
    const size_t want = std::min<size_t>({(nbm ? (size_t)atoi(nbm) : 3) * wbytes, (size_t)max_win, (size_t)max_pers});
    if (want > 0) {
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      cudaStreamAttrValue a{};
      a.accessPolicyWindow.base_ptr = g->bits;
      a.accessPolicyWindow.num_bytes = want;
      a.accessPolicyWindow.hitRatio = 1.0f;
      a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &a);
      cudaGetLastError();  // best effort: persistence is an optimisation only
    }
  }
  return GK_OK;
}

// Kernel parameters of one traversal on g (tuning knobs read from the environment).
gk::BfsParams make_params(gk_graph* g, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy,
                          int want_depth) {
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
  p.parent = g->parent;
  p.depth = g->depth;
  p.visited = g->visited;
  p.dead = g->dead;
  p.head = g->head;
  p.head2 = getenv("GK_NO_HEAD2") ? nullptr : g->head2;
  p.hbase = g->hbase;
  p.live = g->live;
  p.deg16 = g->deg16;
  if (g->own_split && !p.front_in_smem && !getenv("GK_NO_OWN")) {
    p.own_split = g->own_split;
    p.hv_bits = g->hv_bits;
    p.hv_base = g->hv_base;
    p.own_list = g->own_list;
    p.own_stage = g->own_stage;
    p.own_r = g->own_r;
    p.own_span_w = (int32_t)g->own_span_w;
    p.own_win_log = g->own_win_log;
    p.own_dmin = g->own_dmin;
  }
  p.bm0 = g->bm0;
  p.bm1 = g->bm1;
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
  // kTopDownRescan re-reads every new frontier's queue (bfs.hpp:161-167):
  // its steps keep the queue path (large steps leave the frontier a bitmap)
  if (strategy == GK_BFS_TOP_DOWN_RESCAN) p.bitmap_td_min = INT64_MAX;
  p.queue = g->queue;
  p.chunks = g->chunks;
  p.chunk_cap = g->chunk_cap;
  p.ctrl = g->ctrl;
  p.steps = g->steps;
  p.step_cap = g->step_cap;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  if (const char* w = getenv("GK_WATCHDOG_MS")) p.timeout_ns = strtoull(w, nullptr, 10) * 1000000ull;
  p.stop_after = 0xffffffffu;
  if (const char* sa = getenv("GK_STOP_AFTER")) p.stop_after = (unsigned)strtoul(sa, nullptr, 10);

  return p;
}

// Control blocks alternate between launches: each launch zeroes the other
// one during its init phase, so no memset sits between launches.  After a
// failed launch both are cleared (the kernel may not have finished that).
void use_ctrl(gk_graph* g, gk::BfsParams& p) {  // call launched() once the kernel is queued
  p.ctrl = g->ctrl + (g->ctrl_epoch & 1);
  p.ctrl_next = g->ctrl + ((g->ctrl_epoch + 1) & 1);
}
void launched(gk_graph* g) { g->ctrl_epoch++; }
void reset_ctrl(gk_graph* g) {
  cudaMemset(g->ctrl, 0, 2 * sizeof(gk::Ctrl));
  g->ctrl_epoch = 0;
}

gk_status finish_graph(gk_graph* g, gk_graph** out) {
  // every kernel indexes with these arrays: reject a malformed CSR up front
  for (int pass = 0; pass < (g->directed ? 2 : 1); pass++) {
    bool off_ok = true, ids_ok = true;
    const cudaError_t e = gk::validate_csr(pass ? g->in_off : g->out_off, pass ? g->in_nb : g->out_nb, g->n, g->m,
                                           g->n, &off_ok, &ids_ok, nullptr);
    if (e != cudaSuccess || !off_ok || !ids_ok) {
      free_graph(g);
      if (e != cudaSuccess) return cuda_fail(e, "validate CSR");
      return fail(GK_ERR_INVALID, !off_ok ? "invalid graph: offsets not monotone from 0 to m"
                                          : "invalid graph: neighbour id out of range");
    }
  }
  gk_status st = alloc_workspace(g);
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
  if ((e = cudaMalloc(&g->out_off, ob + 16)) || (e = cudaMalloc(&g->out_nb, nbb)) ||
      (e = cudaMemcpy(g->out_off, csr->out_offsets, ob, cudaMemcpyHostToDevice)) ||
      (g->m && (e = cudaMemcpy(g->out_nb, csr->out_neighbors, sizeof(uint32_t) * g->m,
                               cudaMemcpyHostToDevice)))) {
    free_graph(g);
    return cuda_fail(e, "upload CSR");
  }
  if (g->directed) {
    if ((e = cudaMalloc(&g->in_off, ob + 16)) || (e = cudaMalloc(&g->in_nb, nbb)) ||
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

gk_status gk_bfs(gk_graph* g, uint32_t source, int64_t alpha, int64_t beta, int32_t strategy,
                 int32_t* parent_out, int32_t* depth_out, gk_bfs_stats* stats) {
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

  gk::BfsParams p = make_params(g, source, alpha, beta, strategy, want_depth);

  cudaStream_t s = g->stream;
  use_ctrl(g, p);
  CK(cudaEventRecord(g->ev0, s), "event record");
  CK(gk::bfs_launch(p, g->launch, s), "launch bfs kernel");
  launched(g);
  CK(cudaEventRecord(g->ev1, s), "event record");
  gk::Ctrl& ctrl = g->last_ctrl;
  g->last_valid = 0;
  CK(cudaMemcpyAsync(&ctrl, p.ctrl, sizeof(ctrl), cudaMemcpyDeviceToHost, s), "read ctrl");
  CK(cudaStreamSynchronize(s), "bfs kernel");
  g->last_valid = 1;
  g->depth_valid = want_depth;
  if (ctrl.error) {
    reset_ctrl(g);
    if (ctrl.error == 2) {
      unsigned lo = ~0u, hi = 0;
      for (int i = 0; i < 2048; i++) {
        if (ctrl.cta_ph[i] == 0) continue;
        lo = std::min(lo, ctrl.cta_ph[i]);
        hi = std::max(hi, ctrl.cta_ph[i]);
      }
      char buf[256];
      snprintf(buf, sizeof(buf),
               "bfs kernel watchdog fired (grid barrier timeout): CTA barrier counts min %u max %u, "
               "arrivals %llu",
               lo, hi, (unsigned long long)ctrl.bar_count);
      return fail(GK_ERR_TIMEOUT, buf);
    }
    return fail(GK_ERR_CUDA, "bfs kernel: heavy-chunk buffer overflow");
  }
  if (stats) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1), "event time");
    stats->device_ms = ms;
    stats->num_steps = (int32_t)ctrl.num_steps;
    if (stats->steps && stats->max_steps > 0) {
      int64_t k = std::min<int64_t>({(int64_t)stats->max_steps, ctrl.num_steps, g->step_cap});
      if (k > 0)
        CK(cudaMemcpy(stats->steps, g->steps, sizeof(gk_step) * k, cudaMemcpyDeviceToHost), "read steps");
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
  if (parent_out && g->n)
    CK(cudaMemcpyAsync(parent_out, g->parent, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost, s), "D2H parent");
  if (depth_out && g->n)
    CK(cudaMemcpyAsync(depth_out, g->depth, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost, s), "D2H depth");
  if (parent_out || depth_out) CK(cudaStreamSynchronize(s), "D2H");
  return GK_OK;
}

// Many traversals with their parent arrays returned to host memory: the
// D2H copy of traversal i (on a second stream) overlaps traversal i+1 (two
// device parent buffers), so a run is bound by max(kernel, copy) per
// source instead of their sum.  Same validation and results as gk_bfs.
gk_status gk_bfs_batch(gk_graph* g, const uint32_t* sources, int32_t count, int64_t alpha, int64_t beta,
                       int32_t strategy, int32_t* const* parents_out, float* device_ms) {
  if (!g) return fail(GK_ERR_INVALID, "null graph");
  if (count < 0 || (count > 0 && !sources)) return fail(GK_ERR_INVALID, "null argument");
  for (int32_t i = 0; i < count; i++)
    if ((int64_t)sources[i] >= g->n) return fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  if (alpha <= 0 || beta <= 0) return fail(GK_ERR_BAD_PARAM, "bfs alpha and beta must be positive");
  if (strategy < 0 || strategy > 2) return fail(GK_ERR_BAD_PARAM, "unknown bfs strategy");
  if (count == 0) return GK_OK;
  std::lock_guard<std::mutex> lock(g->mu);
  CK(cudaSetDevice(g->device), "cudaSetDevice");
  if (!g->parent2) CK(cudaMalloc(&g->parent2, sizeof(int32_t) * std::max<int64_t>(g->n, 4) + 16), "alloc parent");
  if (!g->cstream) CK(cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking), "stream");
  cudaStream_t s = g->stream, cs = g->cstream;
  std::vector<cudaEvent_t> ev(2 * (size_t)count + 4, nullptr);
  int* errs = nullptr;
  gk_status st = GK_OK;
  auto cleanup = [&]() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (errs) cudaFreeHost(errs);
  };
  for (auto& e : ev)
    if (cudaEventCreate(&e) != cudaSuccess) {
      cleanup();
      return fail(GK_ERR_CUDA, "event create");
    }
  if (cudaHostAlloc(&errs, sizeof(int) * count, cudaHostAllocDefault) != cudaSuccess) {
    cleanup();
    return fail(GK_ERR_CUDA, "cudaHostAlloc");
  }
  cudaEvent_t* kdone = &ev[2 * (size_t)count];  // [2] kernel of slot done
  cudaEvent_t* cdone = kdone + 2;               // [2] copy of slot done
  int32_t* buf[2] = {g->parent, g->parent2};
  g->last_valid = 0;
  g->depth_valid = 0;
  cudaError_t e = cudaSuccess;
  for (int32_t i = 0; i < count && e == cudaSuccess; i++) {
    const int slot = i & 1;
    gk::BfsParams p = make_params(g, sources[i], alpha, beta, strategy, 0);
    p.parent = buf[slot];
    use_ctrl(g, p);
    if (i >= 2 && (e = cudaStreamWaitEvent(s, cdone[slot], 0))) break;  // copy of i-2 has left buf
    if ((e = cudaEventRecord(ev[2 * i], s))) break;
    if ((e = gk::bfs_launch(p, g->launch, s))) break;
    launched(g);
    if ((e = cudaEventRecord(ev[2 * i + 1], s))) break;
    if ((e = cudaMemcpyAsync(errs + i, &p.ctrl->error, sizeof(int), cudaMemcpyDeviceToHost, s))) break;
    if ((e = cudaEventRecord(kdone[slot], s))) break;
    if ((e = cudaStreamWaitEvent(cs, kdone[slot], 0))) break;
    if (parents_out && parents_out[i] &&
        (e = cudaMemcpyAsync(parents_out[i], buf[slot], sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost, cs)))
      break;
    if ((e = cudaEventRecord(cdone[slot], cs))) break;
  }
  cudaError_t e2 = cudaStreamSynchronize(s), e3 = cudaStreamSynchronize(cs);
  if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : e3;
  if (e != cudaSuccess) {
    cleanup();
    reset_ctrl(g);
    return fail(GK_ERR_CUDA, std::string("bfs batch: ") + cudaGetErrorString(e));
  }
  for (int32_t i = 0; i < count; i++)
    if (errs[i]) {
      reset_ctrl(g);
      break;
    }
  for (int32_t i = 0; i < count && st == GK_OK; i++) {
    if (errs[i] == 2) st = fail(GK_ERR_TIMEOUT, "bfs kernel watchdog fired (grid barrier timeout)");
    else if (errs[i]) st = fail(GK_ERR_CUDA, "bfs kernel: heavy-chunk buffer overflow");
    if (device_ms && st == GK_OK) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      device_ms[i] = ms;
    }
  }
  if ((count - 1) & 1) std::swap(g->parent, g->parent2);  // g->parent = the last result
  cleanup();
  return st;
}

const int32_t* gk_bfs_device_parent(const gk_graph* g) { return g ? g->parent : nullptr; }

gk_status gk_bfs_trace(const gk_graph* g, uint64_t* ts_ns, char* tags, int32_t cap, int32_t* count) {
  if (!g || !count) return fail(GK_ERR_INVALID, "null argument");
  if (!g->last_valid) return fail(GK_ERR_INVALID, "no completed gk_bfs on this handle");
  int32_t k = 0;
  for (int32_t i = 0; i < gk::kTraceCap; i++) {
    if (i > 0 && g->last_ctrl.tag[i] == 0) break;
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
// betweenness.hpp:86-93.
gk_status gk_brandes(gk_graph* g, const uint32_t* sources, int64_t num_sources, float* scores_out,
                     double* device_ms) {
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
  if (!g->depth) CK(cudaMalloc(&g->depth, sizeof(int32_t) * std::max<int64_t>(n, 4) + 16), "alloc depth");
  if (!g->bc_sd) {
    CK(cudaMalloc(&g->bc_sd, sizeof(double2) * std::max<int64_t>(n, 1)), "alloc sigma/delta");
    CK(cudaMalloc(&g->bc_succ, sizeof(uint32_t) * ((g->m + 31) / 32 + 1)), "alloc successor bitmap");
    CK(cudaMalloc(&g->bc_scores, sizeof(float) * std::max<int64_t>(n, 1) + 16), "alloc scores");
    g->bc_bounds_cap = n + 2;
    CK(cudaMalloc(&g->bc_bounds, sizeof(int64_t) * g->bc_bounds_cap), "alloc level bounds");
    CK(cudaMalloc(&g->bc_lv, sizeof(uint32_t) * gk::kBcMaxPull * ((n + 31) / 32 + 4)), "alloc level bitmaps");
    CK(cudaMalloc(&g->bc_lvdeg, sizeof(long long) * gk::kBcMaxPull), "alloc level arc sums");
  }
  g->last_valid = 0;  // depth/queue now hold Brandes state
  g->depth_valid = 0;
  gk::BfsParams p{};
  p.n = n;
  p.m = g->m;
  p.w32 = (n + 31) / 32;
  p.out_off = g->out_off;
  p.out_nb = g->out_nb;
  p.in_off = g->in_off;
  p.in_nb = g->in_nb;
  p.depth = g->depth;
  p.queue = g->queue;
  p.chunks = g->chunks;
  p.chunk_cap = g->chunk_cap;
  p.ctrl = g->ctrl;
  p.steps = g->steps;
  p.step_cap = g->step_cap;
  p.timeout_ns = 20ull * 1000 * 1000 * 1000;
  if (const char* w = getenv("GK_WATCHDOG_MS")) p.timeout_ns = strtoull(w, nullptr, 10) * 1000000ull;
  p.stop_after = 0xffffffffu;
  p.bc_sd = g->bc_sd;
  p.bc_succ = g->bc_succ;
  p.bc_scores = g->bc_scores;
  p.bc_bounds = g->bc_bounds;
  p.bc_bounds_cap = g->bc_bounds_cap;
  p.bc_lv = g->bc_lv;
  p.bc_lvw = (n + 31) / 32 + 4;
  p.bc_lvdeg = g->bc_lvdeg;
  p.visited = g->visited;
  p.dead = g->dead;
  p.bm0 = g->bm0;
  if (getenv("GK_BC_NO_PULL")) p.bc_lv = nullptr;  // top-down only (the reference's forward)
  cudaStream_t s = g->stream;
  CK(cudaMemsetAsync(g->bc_scores, 0, sizeof(float) * n, s), "clear scores");
  CK(cudaEventRecord(g->ev0, s), "event record");
  for (int64_t i = 0; i < num_sources; i++) {
    p.src = sources[i];
    use_ctrl(g, p);
    CK(gk::bc_launch(p, g->device, s), "launch brandes kernel");
    launched(g);
    gk::Ctrl& ctrl = g->last_ctrl;  // kept for gk_bfs_trace (phase timings of the last source)
    CK(cudaMemcpyAsync(&ctrl, p.ctrl, sizeof(ctrl), cudaMemcpyDeviceToHost, s), "read ctrl");
    CK(cudaStreamSynchronize(s), "brandes kernel");
    g->last_valid = 1;
    const int err = ctrl.error;
    if (err) reset_ctrl(g);
    if (err == 2) return fail(GK_ERR_TIMEOUT, "brandes kernel watchdog fired (grid barrier timeout)");
    if (err == 3) return fail(GK_ERR_CUDA, "brandes kernel: chunk buffer overflow");
    if (err == 4) return fail(GK_ERR_CUDA, "brandes kernel: level bound buffer overflow");
    if (err) return fail(GK_ERR_CUDA, "brandes kernel failed");
  }
  CK(gk::bc_normalize(g->bc_scores, n, g->bc_scores + n, s), "normalize scores");
  CK(cudaEventRecord(g->ev1, s), "event record");
  if (scores_out) CK(cudaMemcpyAsync(scores_out, g->bc_scores, sizeof(float) * n, cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaStreamSynchronize(s), "brandes");
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
