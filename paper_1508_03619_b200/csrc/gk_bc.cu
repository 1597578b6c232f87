// gk_bc.cu -- Brandes betweenness on the persistent
// BFS machinery: one cooperative launch per source (bc_persistent), then a
// max normalisation.  Restates gapkit::Brandes / detail::BrandesForward
// (proj/include/gapkit/kernels/betweenness.hpp:38-145).
#include <algorithm>

#include "gk_persistent.cuh"

namespace gk {
namespace {

// ============================================================================
// Brandes betweenness (betweenness.hpp:38-80, 84-145), one source per launch.
//
// Forward: level-synchronous top-down BFS that also counts shortest paths
// (sigma, doubles; path counts are integers, so the order of the atomic
// adds does not change them below 2^53) and flags each shortest-path
// successor edge in an m-bit bitmap, exactly the reference's BrandesForward
// (betweenness.hpp:38-80): a target first seen at depth -1 is claimed with a
// CAS; every edge whose target ends up at the current depth sets its
// successor bit and adds sigma[u] into sigma[v].  The queue keeps every
// level in place; bc_bounds[d] marks where level d starts.
// Backward (betweenness.hpp:104-122): levels deepest first; delta[u] = sum
// over u's flagged edges of sigma[u]/sigma[v] * (1 + delta[v]), edge-balanced
// over the level like the forward expansion (per-vertex sums in shared
// memory, high-degree vertices in chunks whose partial sums are added
// atomically).  The summation order differs from the reference's serial
// per-vertex loop, so dependencies agree to rounding (path counts are
// exact).  Finally scores[u] += (float)delta[u] for every reached u !=
// source.
// ============================================================================
constexpr int64_t kBcChunk = 1024;

__device__ __forceinline__ void bc_edges4(const BfsParams& P, const QApp& qa, const double (&su)[4],
                                          const uint32_t (&v)[4], const int64_t (&e)[4], const bool (&ok)[4],
                                          int lvl, uint32_t* buf, int& qcnt) {
  int dv[4];
  bool cl[4];
#pragma unroll
  for (int k = 0; k < 4; k++) dv[k] = ok[k] ? __ldcg(P.depth + v[k]) : -2;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    cl[k] = false;
    if (dv[k] == -1) {  // betweenness.hpp:62-65
      const int old = atomicCAS(P.depth + v[k], -1, lvl);
      cl[k] = old == -1;
      dv[k] = cl[k] ? lvl : old;
      if (cl[k] && P.bc_lv) atomicOr(P.visited + (v[k] >> 5), 1u << (v[k] & 31u));  // for pull steps
    }
  }
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (dv[k] == lvl) {  // betweenness.hpp:66-69
      atomicOr(P.bc_succ + (e[k] >> 5), 1u << (e[k] & 31));
      atomicAdd(&P.bc_sd[v[k]].x, su[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 4; k++) wq_push(P, qa, cl[k], v[k], buf, qcnt);
}

// Forward expansion of queue[qs, qe): tiles of kBlock frontier vertices,
// CTA scan of degrees, load-balanced edge gather; degree > kBcChunk vertices
// become chunks for bc_forward_heavy.
__device__ void bc_forward_light(const BfsParams& P, SmemT& s, unsigned ph, const QApp& qa,
                                 unsigned long long qs, unsigned long long qe, int lvl, int& qcnt) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  unsigned long long* cnt = P.ctrl->cnt[ph & 3];
  for (unsigned long long tile = blockIdx.x;; tile += gridDim.x) {
    const unsigned long long start = qs + tile * (unsigned long long)kBlock;
    if (start >= qe) break;
    const unsigned long long i = start + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, dl = 0;
    double su = 0.0;
    if (i < qe) {
      u = __ldcg(P.queue + i);
      b = offv(P, P.out_off, u);
      su = __ldcg(&P.bc_sd[u].x);
      const int64_t d = offv(P, P.out_off, u + 1) - b;
      if (d > kBcChunk) {
        const int64_t nch = (d + kBcChunk - 1) / kBcChunk;
        const unsigned long long base = atomicAdd(&cnt[kChunkCount], (unsigned long long)nch);
        if ((int64_t)(base + nch) <= P.chunk_cap) {
          for (int64_t c = 0; c < nch; c++) {
            Chunk ch;
            ch.u = u;
            ch.start = b + c * kBcChunk;
            ch.len = (uint32_t)((d - c * kBcChunk) < kBcChunk ? (d - c * kBcChunk) : kBcChunk);
            P.chunks[base + c] = ch;
          }
        } else {
          atomicExch(&P.ctrl->error, 3);
        }
      } else {
        dl = d;
      }
    }
    s.td.t_u[threadIdx.x] = u;
    s.td.t_b[threadIdx.x] = b;
    s.bc_sig[threadIdx.x] = su;
    int64_t tot;
    const int64_t pre = block_exscan(dl, &tot, s);
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kBlock) {
      uint32_t v[4];
      int64_t e[4];
      double sg[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kBlock + threadIdx.x;
        ok[k] = ei < tot;
        v[k] = 0;
        e[k] = 0;
        sg[k] = 0.0;
        if (ok[k]) {
          int lo = 0, hi = kBlock - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.td.t_pre[mid] <= ei) lo = mid;
            else hi = mid - 1;
          }
          e[k] = s.td.t_b[lo] + (ei - s.td.t_pre[lo]);
          v[k] = __ldg(P.out_nb + e[k]);
          sg[k] = s.bc_sig[lo];
        }
      }
      bc_edges4(P, qa, sg, v, e, ok, lvl, buf, qcnt);
    }
    __syncthreads();
  }
}

__device__ void bc_forward_heavy(const BfsParams& P, const QApp& qa, unsigned long long nch, int lvl, SmemT& s,
                                 int& qcnt) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
  for (unsigned long long c = gw; c < nch; c += nw) {
    const Chunk ch = P.chunks[c];
    const double su = __ldcg(&P.bc_sd[ch.u].x);
    const double sg[4] = {su, su, su, su};
    for (uint32_t o = 0; o < ch.len; o += 128) {
      uint32_t v[4];
      int64_t e[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t j = o + lane + 32u * k;
        ok[k] = j < ch.len;
        e[k] = ch.start + j;
        v[k] = ok[k] ? __ldg(P.out_nb + e[k]) : 0u;
      }
      bc_edges4(P, qa, sg, v, e, ok, lvl, buf, qcnt);
    }
  }
}

// sigma[u]/sigma[v] * (1 + delta[v]) for a flagged edge (betweenness.hpp:115)
__device__ __forceinline__ double bc_term(const BfsParams& P, double su, uint32_t v) {
  const double2 sd = __ldcg(P.bc_sd + v);  // sigma and delta in one 16-byte access
  return (su / sd.x) * (1.0 + sd.y);
}

// Backward pass A over one level's vertices queue[b0, b1): tiles of kBlock
// vertices, CTA scan of degrees, load-balanced over the tile's edges with 4
// edges per thread in flight; each flagged edge's term is added into its
// vertex's shared-memory accumulator, written to delta once per tile.
// Vertices of degree > kBcChunk are cut into chunks for pass B (their delta
// stays 0 here and collects the chunk partials).
__device__ void bc_backward_level(const BfsParams& P, SmemT& s, unsigned ph, unsigned long long b0,
                                  unsigned long long b1, const uint32_t* lvb) {
  double* acc = reinterpret_cast<double*>(&s.td.qbuf[0][0]);  // kBlock doubles (qbuf unused here)
  unsigned long long* cnt = P.ctrl->cnt[ph & 3];
  for (unsigned long long tile = blockIdx.x;; tile += gridDim.x) {
    const unsigned long long start = b0 + tile * (unsigned long long)kBlock;
    if (start >= b1) break;
    const unsigned long long i = start + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, dl = 0;
    double su = 0.0;
    bool heavy = false;
    if (i < b1) {
      u = __ldcg(P.queue + i);
      b = offv(P, P.out_off, u);
      su = __ldcg(&P.bc_sd[u].x);
      const int64_t d = offv(P, P.out_off, u + 1) - b;
      if (d > kBcChunk) {
        heavy = true;
        const int64_t nch = (d + kBcChunk - 1) / kBcChunk;
        const unsigned long long base = atomicAdd(&cnt[kChunkCount], (unsigned long long)nch);
        if ((int64_t)(base + nch) <= P.chunk_cap) {
          for (int64_t c = 0; c < nch; c++) {
            Chunk ch;
            ch.u = u;
            ch.start = b + c * kBcChunk;
            ch.len = (uint32_t)((d - c * kBcChunk) < kBcChunk ? (d - c * kBcChunk) : kBcChunk);
            P.chunks[base + c] = ch;
          }
        } else {
          atomicExch(&P.ctrl->error, 3);
        }
      } else {
        dl = d;
      }
    }
    s.td.t_b[threadIdx.x] = b;
    s.bc_sig[threadIdx.x] = su;
    acc[threadIdx.x] = 0.0;
    int64_t tot;
    const int64_t pre = block_exscan(dl, &tot, s);
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kBlock) {
      int64_t e[4];
      int lo[4];
      bool f[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kBlock + threadIdx.x;
        f[k] = false;
        lo[k] = 0;
        e[k] = 0;
        if (ei < tot) {
          int l = 0, h = kBlock - 1;
          while (l < h) {
            const int mid = (l + h + 1) >> 1;
            if (s.td.t_pre[mid] <= ei) l = mid;
            else h = mid - 1;
          }
          lo[k] = l;
          e[k] = s.td.t_b[l] + (ei - s.td.t_pre[l]);
          f[k] = lvb ? true : ((__ldcg(P.bc_succ + (e[k] >> 5)) >> (e[k] & 31)) & 1u);
        }
      }
      uint32_t v[4];
#pragma unroll
      for (int k = 0; k < 4; k++) v[k] = f[k] ? __ldg(P.out_nb + e[k]) : 0u;
      if (lvb) {  // level d+1 was found by a pull step: successor = member of its bitmap
#pragma unroll
        for (int k = 0; k < 4; k++) f[k] = f[k] && ((__ldcg(lvb + (v[k] >> 5)) >> (v[k] & 31u)) & 1u);
      }
      double sv[4], dv[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const double2 sd = f[k] ? __ldcg(P.bc_sd + v[k]) : make_double2(1.0, 0.0);
        sv[k] = sd.x;
        dv[k] = sd.y;
      }
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (f[k]) atomicAdd(acc + lo[k], (s.bc_sig[lo[k]] / sv[k]) * (1.0 + dv[k]));
    }
    __syncthreads();
    if (i < b1 && !heavy) P.bc_sd[u].y = acc[threadIdx.x];
    __syncthreads();
  }
}

// Backward pass B: chunks of the level's high-degree vertices.
__device__ void bc_backward_chunks(const BfsParams& P, unsigned long long nch, const uint32_t* lvb) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
  for (unsigned long long c = gw; c < nch; c += nw) {
    const Chunk ch = P.chunks[c];
    const double su = __ldcg(&P.bc_sd[ch.u].x);
    double acc = 0.0;
    for (uint32_t j = lane; j < ch.len; j += 32) {
      const int64_t e = ch.start + j;
      if (lvb) {
        const uint32_t v = __ldg(P.out_nb + e);
        if ((__ldcg(lvb + (v >> 5)) >> (v & 31u)) & 1u) acc += bc_term(P, su, v);
      } else if ((__ldcg(P.bc_succ + (e >> 5)) >> (e & 31)) & 1u) {
        acc += bc_term(P, su, __ldg(P.out_nb + e));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0 && acc != 0.0) atomicAdd(&P.bc_sd[ch.u].y, acc);
  }
}

// Forward level found bottom-up (§8(f)-4's "TD/BU machinery" for Brandes):
// every unvisited live vertex v sums sigma over ALL its in-neighbours in the
// front (no early exit: sigma needs every shortest-path predecessor); v
// joins the level when it has one.  Tiles of kBlock consecutive vertices,
// CTA scan of the pending vertices' in-degrees, 4 in-edges per thread in
// flight, per-vertex sums in shared memory.  The level's membership goes to
// a bitmap (lv) that the backward pass uses as its successor test; sigma is
// an integer count, so the summation order does not change it.
__device__ void bc_pull_level(const BfsParams& P, SmemT& s, unsigned ph, const QApp& qa, int lvl,
                              const uint32_t* front, uint32_t* lv, int& qcnt, long long& degsum) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  double* acc = s.bc_sig;
  uint32_t* hit = s.td.t_u;
  const long long ntiles = (P.n + kBlock - 1) / kBlock;
  // tiles after the first are claimed dynamically: a tile holding a hub's
  // full in-list must not hold back the CTA's statically assigned others
  unsigned long long* tctr = &P.ctrl->cnt[ph & 3][kTile];
  for (long long tile = blockIdx.x; tile < ntiles;) {
    if (threadIdx.x == 0) s.bcast[1] = gridDim.x + atomicAdd(tctr, 1ull);
    const long long v = tile * kBlock + threadIdx.x;
    bool pend = false;
    uint32_t vis = 0xffffffffu;
    int64_t b = 0, dl = 0;
    if (v < P.n) {
      const long long w = v >> 5;
      vis = __ldcg(P.visited + w) | __ldg(P.dead + w);
      pend = !((vis >> (v & 31)) & 1u);
      if (pend) {
        b = offv(P, P.in_off, v);
        dl = offv(P, P.in_off, v + 1) - b;
      }
    }
    s.td.t_b[threadIdx.x] = b;
    acc[threadIdx.x] = 0.0;
    hit[threadIdx.x] = 0u;
    int64_t tot;
    const int64_t pre = block_exscan(dl, &tot, s);
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kBlock) {
      uint32_t u[4];
      int lo[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kBlock + threadIdx.x;
        ok[k] = ei < tot;
        lo[k] = 0;
        u[k] = 0;
        if (ok[k]) {
          int l = 0, h = kBlock - 1;
          while (l < h) {
            const int mid = (l + h + 1) >> 1;
            if (s.td.t_pre[mid] <= ei) l = mid;
            else h = mid - 1;
          }
          lo[k] = l;
          u[k] = ld_nb(P.in_nb + s.td.t_b[l] + (ei - s.td.t_pre[l]));
        }
      }
      bool f[4];
#pragma unroll
      for (int k = 0; k < 4; k++) f[k] = ok[k] && ((ld_front(front + (u[k] >> 5)) >> (u[k] & 31u)) & 1u);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (f[k]) {
          atomicAdd(acc + lo[k], __ldcg(&P.bc_sd[u[k]].x));
          hit[lo[k]] = 1u;
        }
      }
    }
    __syncthreads();
    const bool got = pend && hit[threadIdx.x];
    if (got) {
      P.depth[v] = lvl;
      P.bc_sd[v].x = acc[threadIdx.x];
      degsum += dl;  // in-degree = the level's share of arcs a pushed backward pass scans
    }
    const unsigned m = __ballot_sync(kFull, got);
    if ((threadIdx.x & 31) == 0 && v < P.n) {  // tiles are word-aligned: one writer per word
      lv[v >> 5] = m;
      if (m) P.visited[v >> 5] = vis | m;
    }
    wq_push(P, qa, got, (uint32_t)v, buf, qcnt);
    __syncthreads();
    tile = (long long)s.bcast[1];
    __syncthreads();
  }
}

// Backward pass for level d pushed from level d+1 (used when d+1 was
// pulled and its in-arcs are fewer than level d's out-arcs, e.g. the level
// after a hub expansion): every v in level d+1 adds (1 + delta(v)) /
// sigma(v) into delta(u) of each in-neighbour u in level d (membership
// bitmap ld); bc_push_finish then scales delta(u) by sigma(u).  Same sum
// as betweenness.hpp:115, sigma(u) factored out.
__device__ void bc_push_level(const BfsParams& P, SmemT& s, unsigned long long b0, unsigned long long b1,
                              const uint32_t* ld) {
  double* tv = s.bc_sig;
  for (unsigned long long tile = blockIdx.x;; tile += gridDim.x) {
    const unsigned long long start = b0 + tile * (unsigned long long)kBlock;
    if (start >= b1) break;
    const unsigned long long i = start + threadIdx.x;
    int64_t b = 0, dl = 0;
    double t = 0.0;
    if (i < b1) {
      const uint32_t v = __ldcg(P.queue + i);
      b = offv(P, P.in_off, v);
      dl = offv(P, P.in_off, v + 1) - b;
      const double2 sd = __ldcg(P.bc_sd + v);
      t = (1.0 + sd.y) / sd.x;
    }
    s.td.t_b[threadIdx.x] = b;
    tv[threadIdx.x] = t;
    int64_t tot;
    const int64_t pre = block_exscan(dl, &tot, s);
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kBlock) {
      uint32_t u[4];
      int lo[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kBlock + threadIdx.x;
        ok[k] = ei < tot;
        lo[k] = 0;
        u[k] = 0;
        if (ok[k]) {
          int l = 0, h = kBlock - 1;
          while (l < h) {
            const int mid = (l + h + 1) >> 1;
            if (s.td.t_pre[mid] <= ei) l = mid;
            else h = mid - 1;
          }
          lo[k] = l;
          u[k] = ld_nb(P.in_nb + s.td.t_b[l] + (ei - s.td.t_pre[l]));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (ok[k] && ((ld_front(ld + (u[k] >> 5)) >> (u[k] & 31u)) & 1u)) atomicAdd(&P.bc_sd[u[k]].y, tv[lo[k]]);
    }
    __syncthreads();
  }
}

__device__ void bc_push_finish(const BfsParams& P, unsigned long long b0, unsigned long long b1) {
  for (unsigned long long i = b0 + (unsigned long long)blockIdx.x * kBlock + threadIdx.x; i < b1;
       i += (unsigned long long)gridDim.x * kBlock) {
    const uint32_t u = __ldcg(P.queue + i);
    const double2 sd = __ldcg(P.bc_sd + u);
    P.bc_sd[u].y = sd.x * sd.y;
  }
}

__global__ void __launch_bounds__(kBlock, 2) bc_persistent(BfsParams P) {
  __shared__ SmemT s;
  unsigned ph = 0;
  const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gthreads = (long long)gridDim.x * kBlock;
  const uint32_t src = P.src;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->ts[0] = globaltimer();
  // init (betweenness.hpp:96-101)
  for (long long i = gtid; i < P.n; i += gthreads) {
    P.depth[i] = -1;
    P.bc_sd[i] = make_double2(0.0, 0.0);
  }
  const long long sw = (P.m + 31) >> 5;
  for (long long i = gtid; i < sw; i += gthreads) P.bc_succ[i] = 0u;
  if (P.bc_lv)
    for (long long i = gtid; i < P.w32; i += gthreads) P.visited[i] = __ldg(P.dead + i);
  if (!grid_sync(P, s, ph, kTagInit)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // betweenness.hpp:44-48
    P.depth[src] = 0;
    P.bc_sd[src].x = 1.0;
    P.queue[0] = src;
    P.bc_bounds[0] = 0;
    if (P.bc_lv) P.visited[src >> 5] |= 1u << (src & 31u);
  }
  if (!grid_sync(P, s, ph, kTagInit)) return;
  unsigned long long qs = 0, qe = 1, qtail = 1;
  int lvl = 0;
  int qcnt = 0;
  int npull = 0;
  const uint32_t* prev_lv = nullptr;  // bitmap of the previous level when it was pulled
  long long nvis = 1;
  constexpr long long kBcPullRatio = 15;  // pull when the frontier exceeds 1/15 of the unvisited ids
  while (qe > qs) {  // forward levels
    lvl++;
    if (lvl + 1 >= P.bc_bounds_cap) {
      if (threadIdx.x == 0) atomicExch(&P.ctrl->error, 4);
      return;
    }
    const long long fsize = (long long)(qe - qs);
    bool pull = P.bc_lv && npull < kBcMaxPull && fsize * kBcPullRatio > P.n - nvis;
    if (P.bc_lv && npull < kBcMaxPull && !pull && fsize > kBlock) {
      // a few high-degree vertices can hold most edges: decide by the
      // frontier's degree sum against the arcs (BFS's alpha rule, bfs.hpp:144)
      long long dsum = 0;
      for (unsigned long long i = qs + gtid; i < qe; i += gthreads) {
        const uint32_t u = __ldcg(P.queue + i);
        dsum += offv(P, P.out_off, u + 1) - offv(P, P.out_off, u);
      }
      const unsigned set = ph & 3;
      block_add(dsum, &P.ctrl->cnt[set][kSum], s);
      if (!grid_sync(P, s, ph, kTagRescan)) return;
      pull = (long long)s.snap[kSum] * kBcPullRatio > P.m;
    }
    int64_t tag = 0;
    if (pull) {
      const uint32_t* front = prev_lv;
      if (!front) {  // QueueToBitmap of the previous (top-down) level
        for (long long i = gtid; i < P.w32; i += gthreads) P.bm0[i] = 0u;
        if (!grid_sync(P, s, ph, kTagZero)) return;
        for (unsigned long long i = qs + gtid; i < qe; i += gthreads) {
          const uint32_t u = __ldcg(P.queue + i);
          atomicOr(P.bm0 + (u >> 5), 1u << (u & 31u));
        }
        if (!grid_sync(P, s, ph, kTagQ2B)) return;
        front = P.bm0;
      }
      uint32_t* lv = P.bc_lv + (int64_t)npull * P.bc_lvw;
      const QApp qa = qapp(P, ph, qtail);
      long long degsum = 0;
      const unsigned set = ph & 3;
      bc_pull_level(P, s, ph, qa, lvl, front, lv, qcnt, degsum);
      wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
      block_add(degsum, &P.ctrl->cnt[set][kSum], s);
      if (!grid_sync(P, s, ph, kTagBU)) return;
      qtail += s.snap[kAppend];
      if (blockIdx.x == 0 && threadIdx.x == 0) P.bc_lvdeg[npull] = (long long)s.snap[kSum];
      tag = (int64_t)(npull + 1) << 56;
      prev_lv = lv;
      npull++;
    } else {
      {
        const QApp qa = qapp(P, ph, qtail);
        bc_forward_light(P, s, ph, qa, qs, qe, lvl, qcnt);
        wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
      }
      if (!grid_sync(P, s, ph, kTagTD)) return;
      qtail += s.snap[kAppend];
      const unsigned long long nch = s.snap[kChunkCount];
      if (nch) {
        const QApp qa = qapp(P, ph, qtail);
        bc_forward_heavy(P, qa, nch, lvl, s, qcnt);
        wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
        if (!grid_sync(P, s, ph, kTagHeavy)) return;
        qtail += s.snap[kAppend];
      }
      prev_lv = nullptr;
    }
    // level lvl starts at qe
    if (blockIdx.x == 0 && threadIdx.x == 0) P.bc_bounds[lvl] = (int64_t)qe | tag;
    nvis += (long long)(qtail - qe);
    qs = qe;
    qe = qtail;
  }
  // levels 0 .. lvl-1: level d = [bounds[d], bounds[d+1]), bounds[lvl] = qtail
  constexpr int64_t kPosMask = (int64_t(1) << 56) - 1;
  for (int d = lvl - 1; d >= 0; d--) {
    // bounds[lvl] (the empty last level) was written by CTA 0 after the last
    // barrier: never read it -- level lvl has no vertices, so no successors
    const int64_t bd = d == 0 ? 0 : __ldcg(P.bc_bounds + d);
    const int64_t bn = d + 1 == lvl ? 0 : __ldcg(P.bc_bounds + d + 1);
    const unsigned long long b0 = (unsigned long long)(bd & kPosMask);
    const unsigned long long b1 = d + 1 == lvl ? qtail : (unsigned long long)(bn & kPosMask);
    const int pk = (int)((unsigned long long)bn >> 56);  // level d+1 pulled: its bitmap is the successor test
    const uint32_t* lvb = pk ? P.bc_lv + (int64_t)(pk - 1) * P.bc_lvw : nullptr;
    if (pk) {
      // level d+1 was pulled: push from it when its in-arcs are fewer than
      // level d's out-arcs
      const unsigned long long b2 = d + 2 == lvl ? qtail : (unsigned long long)(__ldcg(P.bc_bounds + d + 2) & kPosMask);
      const int pkd = (int)((unsigned long long)bd >> 56);
      long long out_d;
      if (pkd) {
        out_d = __ldcg(P.bc_lvdeg + pkd - 1);
      } else {  // degree sum of level d (top-down): one pass over its queue range
        long long sum = 0;
        for (unsigned long long i = b0 + gtid; i < b1; i += gthreads) {
          const uint32_t u = __ldcg(P.queue + i);
          sum += offv(P, P.out_off, u + 1) - offv(P, P.out_off, u);
        }
        const unsigned set = ph & 3;
        block_add(sum, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagRescan)) return;
        out_d = (long long)s.snap[kSum];
      }
      if (__ldcg(P.bc_lvdeg + pk - 1) < out_d) {
        const uint32_t* ldm = pkd ? P.bc_lv + (int64_t)(pkd - 1) * P.bc_lvw : P.bm0;
        if (!pkd) {  // membership bitmap of level d
          for (long long i = gtid; i < P.w32; i += gthreads) P.bm0[i] = 0u;
          if (!grid_sync(P, s, ph, kTagZero)) return;
          for (unsigned long long i = b0 + gtid; i < b1; i += gthreads) {
            const uint32_t u = __ldcg(P.queue + i);
            atomicOr(P.bm0 + (u >> 5), 1u << (u & 31u));
          }
          if (!grid_sync(P, s, ph, kTagQ2B)) return;
        }
        bc_push_level(P, s, b1, b2, ldm);
        if (!grid_sync(P, s, ph, kTagBcBack)) return;
        bc_push_finish(P, b0, b1);
        if (!grid_sync(P, s, ph, kTagBcChunk)) return;
        continue;
      }
    }
    bc_backward_level(P, s, ph, b0, b1, lvb);
    if (!grid_sync(P, s, ph, kTagBcBack)) return;
    const unsigned long long nch = s.snap[kChunkCount];
    if (nch) {
      bc_backward_chunks(P, nch, lvb);
      if (!grid_sync(P, s, ph, kTagBcChunk)) return;
    }
  }
  // betweenness.hpp:118-119
  for (unsigned long long i = gtid; i < qtail; i += gthreads) {
    const uint32_t u = __ldcg(P.queue + i);
    if (u != src) P.bc_scores[u] += static_cast<float>(__ldcg(&P.bc_sd[u].y));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->num_steps = lvl;
}

__global__ void k_bc_max(const float* __restrict__ x, int64_t n, float* out) {
  float m = 0.0f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, x[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  // scores are >= 0, so the float bit pattern orders like an unsigned int
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned*>(out), __float_as_uint(m));
}
__global__ void k_bc_scale(float* __restrict__ x, int64_t n, const float* mx) {
  const float m = *mx;
  if (!(m > 0.0f)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] /= m;
}

}  // namespace

cudaError_t bc_launch(const BfsParams& p, int device, cudaStream_t st) {
  cudaError_t e;
  int sms = 0, occ = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bc_persistent, kBlock, 0))) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  if ((e = cudaMemsetAsync(p.ctrl, 0, kCtrlClear, st))) return e;
  BfsParams local = p;
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel((const void*)bc_persistent, dim3(sms * occ), dim3(kBlock), args, 0, st);
}

cudaError_t bc_normalize(float* scores, int64_t n, float* scratch_max, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(scratch_max, 0, sizeof(float), st))) return e;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
  k_bc_max<<<grid, 256, 0, st>>>(scores, n, scratch_max);
  k_bc_scale<<<grid, 256, 0, st>>>(scores, n, scratch_max);
  return cudaGetLastError();
}

}  // namespace gk
