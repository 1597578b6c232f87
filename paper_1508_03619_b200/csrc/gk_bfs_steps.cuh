// gk_bfs_steps.cuh -- the phases of the persistent direction-optimizing BFS
// (top-down tiles / heavy chunks / owned-range hubs / claim sweep,
// bottom-up sweep / long lists / sparse sweeps, BitmapToQueue), shared by
// the single-device kernel (gk_bfs_kernel.cu) and the sharded one
// (gk_bfs_sharded.cu).  Every phase works on its rank's part of the launch
// (cta_id / cta_count, owned words [w_lo, w_hi), rank counter sets), which
// for a single-device traversal is the whole grid and the whole bitmap.
// Internal linkage: each kernel file compiles its own copy.
#pragma once

#include "gk_persistent.cuh"

#ifndef GK_SHARDED_STEPS
#define GK_SHARDED_STEPS 0  // 1 in gk_bfs_sharded.cu (compile-time: the single-device kernel pays nothing)
#endif

#ifndef GK_HEAVY_KE
#define GK_HEAVY_KE 8  // heavy-chunk edges per lane in flight (large steps)
#endif

namespace gk {
namespace {

// Parent slot of a claimed vertex: this traversal's array, or -- sharded --
// the owner's (a peer's array when v is remote: the store crosses NVLink,
// fire-and-forget like every bitmap claim; racing claimers store valid
// parents).
__device__ __forceinline__ int32_t* parent_slot(const BfsParams& P, uint32_t v) {
  if constexpr (GK_SHARDED_STEPS) {
    // owner = v / shard_block by a multiply-high with the host's reciprocal
    // (shard_recip = ceil(2^32 / block)), corrected by one step either way
    uint32_t q = __umulhi(v, P.shard_recip);
    const uint32_t b = (uint32_t)P.shard_block;
    if (q * b > v) q--;
    else if ((q + 1) * b <= v) q++;
    return P.shard_parent[q] + v;
  }
  return P.parent + v;
}

__device__ __forceinline__ void on_claim(const BfsParams& P, uint32_t u, uint32_t v, int lvl,
                                         bool encode, long long& scout) {
  P.parent[v] = (int32_t)u;
  if (P.want_depth) P.depth[v] = lvl + 1;
  if (encode) {
    long long d = offv(P, P.out_off, v + 1) - offv(P, P.out_off, v);
    scout += d ? d : 1;  // -old of the degree-encoded slot (bfs.hpp:83,130)
  } else {
    scout += 1;  // unencoded slot is -1 (bfs.hpp:129-130 with encode off)
  }
}

// Claim up to 4 edges (u_k -> v_k) per thread with their loads and atomics
// issued together (bfs.hpp:77-84).  The visited word is read from L2 first
// so already-visited targets cost no atomic.  kBig (large frontiers): the
// claims go only into the next-frontier bitmap (a following bottom-up step
// needs no QueueToBitmap, a following top-down step converts it with
// BitmapToQueue), and their degrees are summed afterwards by td_scout_bits
// in vertex order instead of by random reads at claim time.
template <bool kBig>
__device__ __forceinline__ void claim4(const BfsParams& P, const QApp& qa, const uint32_t (&u)[4],
                                       const uint32_t (&v)[4], const bool (&ok)[4],
                                       uint32_t* nextbm, int lvl, bool encode, long long& scout,
                                       uint32_t* buf, int& qcnt, bool tiny, uint32_t rlo = 0,
                                       uint32_t rhi = 0xffffffffu) {
  uint32_t w[4];
  bool c[4];
  if (!kBig && tiny) {
    // Tiny steps are latency chains (one grid barrier each on high-diameter
    // graphs): no L2 pre-check, and the degree reads go out together with
    // the claim atomics instead of after them.
    int64_t o0[4], o1[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      o0[k] = o1[k] = 0;
      if (ok[k] && encode) {
        o0[k] = offv(P, P.out_off, v[k]);
        o1[k] = offv(P, P.out_off, v[k] + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t bit = 1u << (v[k] & 31u);
      c[k] = ok[k] && !(atomicOr(P.visited + (v[k] >> 5), bit) & bit);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (c[k]) {
        P.parent[v[k]] = (int32_t)u[k];
        if (P.want_depth) P.depth[v[k]] = lvl + 1;
        const long long d = o1[k] - o0[k];
        scout += encode ? (d ? d : 1) : 1;
        // the next level reads this list: start pulling it toward L2 now
        if (encode && d) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.out_nb + o0[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) wq_push(P, qa, c[k], v[k], buf, qcnt);
    return;
  }
  if constexpr (kBig) {
    // Fire-and-forget claims: the next-frontier bitmap starts as a copy of
    // visited, so one pre-check covers both "already visited" and "already
    // claimed this step"; racing writers all store a valid parent (any
    // frontier neighbour) and OR the same bit.  td_scout_bits strips the
    // visited bits afterwards.  No atomic round trip sits on the chain.
    uint32_t x[4];
#pragma unroll
    for (int k = 0; k < 4; k++)
      x[k] = (ok[k] && v[k] >= rlo && v[k] < rhi) ? ld_bits(nextbm + (v[k] >> 5)) : 0xffffffffu;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (!((x[k] >> (v[k] & 31u)) & 1u)) {
#ifndef GK_TD_NO_PARENT  // diagnostic A/B only (results invalid without it)
        st_parent(parent_slot(P, v[k]), (int32_t)u[k]);
#endif
        atomicOr(nextbm + (v[k] >> 5), 1u << (v[k] & 31u));  // result unused -> RED
      }
    }
    return;
  } else {
#pragma unroll
  for (int k = 0; k < 4; k++) w[k] = ok[k] ? ld_bits_l1(P.visited + (v[k] >> 5)) : 0xffffffffu;
#pragma unroll
  for (int k = 0; k < 4; k++) c[k] = !((w[k] >> (v[k] & 31u)) & 1u);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (c[k]) {
      const uint32_t bit = 1u << (v[k] & 31u);
      c[k] = (atomicOr(P.visited + (v[k] >> 5), bit) & bit) == 0;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (c[k]) on_claim(P, u[k], v[k], lvl, encode, scout);
#pragma unroll
  for (int k = 0; k < 4; k++) wq_push(P, qa, c[k], v[k], buf, qcnt);
  }
}

// ---- top-down, light vertices + chunk registration ------------------------
template <bool kBig>
__device__ void td_light(const BfsParams& P, SmemT& s, unsigned ph, const QApp& qa, unsigned long long qs,
                         unsigned long long qe, uint32_t* nextbm, int lvl, bool encode,
                         long long& scout, int& qcnt, int tile_sz, int64_t chunk, bool tiny,
                         bool reg = true, uint32_t rlo = 0, uint32_t rhi = 0xffffffffu, bool own = false) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  unsigned long long* cnt = rset(P, ph);
  // First tile of each CTA is static (no atomic on the latency chain of
  // small levels); the rest are handed out dynamically.
  unsigned long long tile = cta_id(P);
  for (;;) {
    const unsigned long long start = qs + tile * (unsigned long long)tile_sz;
    if (start >= qe) break;
    const unsigned long long i = start + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, dl = 0;
    if ((int)threadIdx.x < tile_sz && i < qe) {
      u = __ldcg(P.queue + i);
      b = offv(P, P.out_off, u);
      const int64_t d = offv(P, P.out_off, u + 1) - b;
      if (own && d >= P.own_dmin) {  // expanded range by range in td_own
        OwnEnt e;
        e.u = u;
        e.deg = (uint32_t)d;
        e.base = b;
        const unsigned long long at = atomicAdd(&cnt[kOwnCount], 1ull);
        if (GK_SHARDED_STEPS) atomicAdd(&P.ctrl->cnt[ph & 3][kWork], 1ull);
        if ((int64_t)at < P.own_cap) P.own_list[at] = e;
        else atomicExch(&P.ctrl->error, 3);  // cannot happen: own_cap >= m / own_dmin
      } else if (d > chunk) {
        if (reg) {  // range passes after the first reuse the chunk list
          const int64_t nch = (d + chunk - 1) / chunk;
          const unsigned long long base = atomicAdd(&cnt[kChunkCount], (unsigned long long)nch);
          if (GK_SHARDED_STEPS) atomicAdd(&P.ctrl->cnt[ph & 3][kWork], 1ull);
          if ((int64_t)(base + nch) <= P.chunk_cap) {
            for (int64_t c = 0; c < nch; c++) {
              Chunk ch;
              ch.u = u;
              ch.start = b + c * chunk;
              ch.len = (uint32_t)((d - c * chunk) < chunk ? (d - c * chunk) : chunk);
              P.chunks[base + c] = ch;
            }
          } else {
            atomicExch(&P.ctrl->error, 3);
          }
        }
      } else {
        dl = d;
      }
    }
    s.td.t_u[threadIdx.x] = u;
    s.td.t_b[threadIdx.x] = b;
    int64_t tot;
    const int64_t pre = block_exscan(dl, &tot, s);
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kBlock) {
      uint32_t uu[4], v[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kBlock + threadIdx.x;
        ok[k] = ei < tot;
        uu[k] = 0;
        v[k] = 0;
        if (ok[k]) {
          int lo = 0, hi = kBlock - 1;  // last item with t_pre <= ei
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.td.t_pre[mid] <= ei) lo = mid;
            else hi = mid - 1;
          }
          uu[k] = s.td.t_u[lo];
          v[k] = ld_nb_once(P.out_nb + s.td.t_b[lo] + (ei - s.td.t_pre[lo]));
        }
      }
      claim4<kBig>(P, qa, uu, v, ok, nextbm, lvl, encode, scout, buf, qcnt, tiny, rlo, rhi);
    }
    // Dynamic tiles only exist past the first gridDim.x; when there are no
    // more tiles than CTAs, nobody pays the fetch-add round trip.
    const bool more = qs + (unsigned long long)cta_count(P) * tile_sz < qe && start + tile_sz < qe;
    if (threadIdx.x == 0 && more) s.bcast[1] = cta_count(P) + atomicAdd(&cnt[kTile], 1ull);
    __syncthreads();
    if (!more) break;  // every later tile starts past qe too
    tile = s.bcast[1];
    __syncthreads();
  }
}

// ---- top-down, heavy chunks: one warp per chunk, 4 edges per lane in flight --
template <bool kBig>
__device__ void td_heavy(const BfsParams& P, SmemT& s, unsigned ph, const QApp& qa, unsigned long long nch,
                         uint32_t* nextbm, int lvl, bool encode, long long& scout, int& qcnt, bool tiny,
                         uint32_t rlo = 0, uint32_t rhi = 0xffffffffu) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  // Chunks are equal-sized (chunk edges but the tails), so a static
  // round-robin over warps balances without a contended grab counter.
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  if constexpr (kBig) {
    // 8 edges per lane in flight and the next chunk descriptor prefetched:
    // the hub step is bound by the nb -> bitmap-word dependent latency
    constexpr int kE = GK_HEAVY_KE;
    // first chunk static, later ones claimed dynamically; the next claim and
    // its descriptor load are issued before the current chunk's edges
    unsigned long long* cctr = &rset(P, ph)[kChunkNext];
    Chunk ch = gw < (long long)nch ? P.chunks[gw] : Chunk{};
    for (unsigned long long c = gw; c < nch;) {
      unsigned long long cn = 0;
      if (lane == 0) cn = nw + atomicAdd(cctr, 1ull);
      cn = __shfl_sync(kFull, cn, 0);
      const Chunk chn = cn < nch ? P.chunks[cn] : Chunk{};
      for (uint32_t o = 0; o < ch.len; o += 32 * kE) {
        uint32_t v[kE], x[kE];
#pragma unroll
        for (int k = 0; k < kE; k++) {
          const uint32_t j = o + lane + 32u * k;
          v[k] = j < ch.len ? ld_nb_once(P.out_nb + ch.start + j) : kNoVertex;
        }
#pragma unroll
        for (int k = 0; k < kE; k++)
          x[k] = (v[k] != kNoVertex && v[k] >= rlo && v[k] < rhi) ? ld_bits(nextbm + (v[k] >> 5)) : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < kE; k++) {
          if (!((x[k] >> (v[k] & 31u)) & 1u)) {  // see claim4<true>
            st_parent(parent_slot(P, v[k]), (int32_t)ch.u);
            atomicOr(nextbm + (v[k] >> 5), 1u << (v[k] & 31u));
          }
        }
      }
      ch = chn;
      c = cn;
    }
    return;
  } else {
  for (unsigned long long c = gw; c < nch; c += nw) {
    const Chunk ch = P.chunks[c];
    const uint32_t uu[4] = {ch.u, ch.u, ch.u, ch.u};
    for (uint32_t o = 0; o < ch.len; o += 128) {
      uint32_t v[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t j = o + lane + 32u * k;
        ok[k] = j < ch.len;
        v[k] = ok[k] ? ld_nb_once(P.out_nb + ch.start + j) : 0u;
      }
      claim4<kBig>(P, qa, uu, v, ok, nextbm, lvl, encode, scout, buf, qcnt, tiny);
    }
  }
  }
}

// ---- top-down, hubs by owned target range ---------------------------------
// The large step's hubs (out-degree >= own_dmin, listed by td_light) are
// expanded range by range: CTA r takes, of every listed hub, the run of its
// ascending out-list whose targets fall in r's id range (the split row gives
// the bounds) and claims them against its slice of the next bitmap held in
// shared memory: a shared-memory test per arc instead of an L2 lookup, and
// exactly one winner per vertex.  Winners are logged per window of
// own_span_w ids; after the runs, each window's parents are gathered in
// shared memory and stored in vertex order (coalesced) -- random 4-byte
// parent stores cost a DRAM sector read-modify-write each (profiles/r01
// random_store_order.txt: 23 vs ~100 G stores/s sorted).  The slice is OR-ed
// back because chunk claims of other CTAs may land in it meanwhile.
#ifndef GK_OWN_KE
#define GK_OWN_KE 12  // 4: -1.2%, 8: -0.3% on kron27
#endif

// Lower bounds of key0 < key1 in the strictly ascending list a[0..d) of ids
// in [0, n): *r0 / *r1 = first index whose id is >= key0 / key1.  A
// bracket (lo, hi) with a[lo] < key <= a[hi] (virtual ends -1 and d)
// shrinks by rounds of three concurrent probes around the interpolated
// position (g - m, g, g + m; m = 2 + 2 sqrt(width)): ids of a permuted graph
// are uniform, so the bracket holds the answer and the width drops to about
// 2 sqrt(width) per round -- 2-3 rounds from a 10^6-arc list to a binary
// search inside one or two cache lines.  Both searches advance together
// (their loads overlap).  Any id distribution terminates with the exact
// answer: a round only ever narrows a valid bracket.
struct SplitSearch {
  int64_t lo, hi;    // a[lo] < key <= a[hi]
  uint32_t vlo, vhi; // ids strictly inside the bracket lie in [vlo, vhi)
  uint32_t key;
};
__device__ __forceinline__ void split_init(SplitSearch& q, uint32_t d, uint32_t key, uint32_t n) {
  q.key = key;
  q.lo = -1;
  q.hi = d;
  q.vlo = 0;
  q.vhi = n;
  if (key == 0) q.hi = 0;        // answer 0
  else if (key >= n) q.lo = (int64_t)d - 1;  // answer d
}
__device__ __forceinline__ int64_t split_width(const SplitSearch& q) { return q.hi - q.lo - 1; }
__device__ __forceinline__ void split_probe_pos(const SplitSearch& q, int64_t& p0, int64_t& p1, int64_t& p2) {
  const int64_t w = split_width(q);
  // interpolated position; float is exact enough (the bracket absorbs it)
  const float f = (float)(q.key - q.vlo) / (float)(q.vhi > q.vlo ? q.vhi - q.vlo : 1u);
  int64_t g = q.lo + 1 + (int64_t)(f * (float)w);
  if (g > q.hi - 1) g = q.hi - 1;
  if (g < q.lo + 1) g = q.lo + 1;
  const int64_t m = 2 + 2 * (int64_t)sqrtf((float)w);
  p0 = g - m > q.lo + 1 ? g - m : q.lo + 1;
  p1 = g;
  p2 = g + m < q.hi - 1 ? g + m : q.hi - 1;
}
__device__ __forceinline__ void split_update(SplitSearch& q, int64_t p0, int64_t p1, int64_t p2, uint32_t x0,
                                             uint32_t x1, uint32_t x2) {
  if (x2 < q.key) {
    q.lo = p2;
    q.vlo = x2 + 1;
  } else if (x1 < q.key) {
    q.lo = p1;
    q.vlo = x1 + 1;
    q.hi = p2;
    q.vhi = x2;
  } else if (x0 < q.key) {
    q.lo = p0;
    q.vlo = x0 + 1;
    q.hi = p1;
    q.vhi = x1;
  } else {
    q.hi = p0;
    q.vhi = x0;
  }
}
__device__ __forceinline__ void split_run(const uint32_t* a, uint32_t d, uint32_t key0, uint32_t key1, uint32_t n,
                                          uint32_t& r0, uint32_t& r1) {
  SplitSearch q[2];
  split_init(q[0], d, key0, n);
  split_init(q[1], d, key1, n);
  constexpr int64_t kBin = 32;  // bracket width finished by binary search (1-2 cache lines)
#pragma unroll 1
  for (int round = 0; round < 4; round++) {
    const bool a0 = split_width(q[0]) > kBin, a1 = split_width(q[1]) > kBin;
    if (!a0 && !a1) break;
    int64_t p[2][3];
    uint32_t x[2][3];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      if (k ? a1 : a0) split_probe_pos(q[k], p[k][0], p[k][1], p[k][2]);
#pragma unroll
      for (int j = 0; j < 3; j++) x[k][j] = (k ? a1 : a0) ? __ldg(a + p[k][j]) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 2; k++)
      if (k ? a1 : a0) split_update(q[k], p[k][0], p[k][1], p[k][2], x[k][0], x[k][1], x[k][2]);
  }
#pragma unroll
  for (int k = 0; k < 2; k++) {
    int64_t lo = q[k].lo, hi = q[k].hi;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(a + mid) < q[k].key) lo = mid;
      else hi = mid;
    }
    (k ? r1 : r0) = (uint32_t)hi;
  }
}

#ifndef GK_OWN_TRACE
#define GK_OWN_TRACE 0  // diagnostics: CTA 0 stamps td_own's sub-phases into ctrl->ts[400..]
#endif
#if GK_OWN_TRACE
#define OWN_MARK(i)                                                                      \
  do {                                                                                   \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                           \
      P.ctrl->ts[400 + (i)] = globaltimer();                                             \
      P.ctrl->tag[400 + (i)] = 'o';                                                      \
    }                                                                                    \
  } while (0)
#else
#define OWN_MARK(i) \
  do {              \
  } while (0)
#endif
__device__ void td_own(const BfsParams& P, SmemT& s, unsigned long long nown, uint32_t* nextbm, uint32_t* sm) {
  OWN_MARK(0);
  constexpr int kE = GK_OWN_KE;  // arcs per lane in flight
  const int r = cta_id(P);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const int sw = P.own_span_w;  // words per range
  const int wlog = P.own_win_log;  // ids per window = 2^wlog <= sw (a shift, not a divide, per claim)
  const int nwin = (32 * sw + (1 << wlog) - 1) >> wlog;  // <= kOwnWin
  const long long w0 = (long long)r * sw;
  const long long w1 = w0 + sw < P.w32 ? w0 + sw : P.w32;
  const int nw = w1 > w0 ? (int)(w1 - w0) : 0;
  uint2* stage = P.own_stage + (int64_t)r * ((int64_t)nwin << wlog);
  const uint32_t key0 = (uint32_t)(w0 * 32);
  const uint32_t key1 = (uint32_t)(w1 * 32 < P.n ? w1 * 32 : P.n);
  for (int i = threadIdx.x; i < nw; i += kBlock) sm[i] = ld_bits(nextbm + w0 + i);
  if (threadIdx.x < kOwnWin) s.own_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (unsigned long long g0 = 0; g0 < nown; g0 += kBlock) {
    // up to kBlock hubs: their runs in this range, concatenated
    const unsigned long long i = g0 + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, len = 0;
    if (i < nown) {
      const OwnEnt e = P.own_list[i];
      uint32_t s0, s1;  // this range's run of the hub's ascending list
      split_run(P.out_nb + e.base, e.deg, key0, key1, (uint32_t)P.n, s0, s1);
      u = e.u;
      b = e.base + s0;
      len = (int64_t)s1 - s0;
    }
    if (g0 == 0) OWN_MARK(1);
    int64_t tot;
    const int64_t pre = block_exscan(len, &tot, s);
    if (g0 == 0) OWN_MARK(2);
    s.td.t_u[threadIdx.x] = u;
    s.td.t_b[threadIdx.x] = b - pre;  // arc of concatenated position e is t_b[o] + e
    s.td.t_pre[threadIdx.x] = pre;
    __syncthreads();
    // Each warp takes a contiguous segment, lanes on consecutive positions
    // (coalesced), and advances its run index as the positions cross run
    // starts -- no per-arc search.  Positions within a group, ids within the
    // range and log indices are 32-bit (fewer live registers in the loop).
    const int tot32 = (int)tot;
    const int seg = ((tot32 + kWarps - 1) / kWarps + 31) & ~31;
    const int eb = (int)warp * seg;
    const int ee = eb + seg < tot32 ? eb + seg : tot32;
    if (eb < ee) {
      int lo = 0, hi = kBlock - 1;  // run holding position eb + lane (clamped)
      const int e0 = eb + (int)lane < ee ? eb + (int)lane : ee - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s.td.t_pre[mid] <= e0) lo = mid;
        else hi = mid - 1;
      }
      int o = lo;
      int nxt = o + 1 < kBlock ? (int)s.td.t_pre[o + 1] : tot32;
      const uint32_t* rb = P.out_nb + s.td.t_b[o];  // arc of position e is rb[e]
      uint32_t ou = s.td.t_u[o];
      const uint32_t id0 = (uint32_t)(w0 * 32);
      const uint32_t wmask = (1u << wlog) - 1u;
      for (int e = eb + (int)lane; e - (int)lane < ee; e += 32 * kE) {
        uint32_t v[kE], uu[kE];
#pragma unroll
        for (int k = 0; k < kE; k++) {
          const int ek = e + 32 * k;
          v[k] = kNoVertex;
          uu[k] = 0;
          if (ek < ee) {
            while (ek >= nxt) {
              o++;
              nxt = o + 1 < kBlock ? (int)s.td.t_pre[o + 1] : tot32;
              rb = P.out_nb + s.td.t_b[o];
              ou = s.td.t_u[o];
            }
            v[k] = ld_nb_once(rb + ek);
            uu[k] = ou;
          }
        }
#pragma unroll
        for (int k = 0; k < kE; k++) {
          if (v[k] == kNoVertex) continue;
          const uint32_t vl = v[k] - id0;  // id within the range
          const uint32_t wl = vl >> 5, bit = 1u << (vl & 31u);
          if (!(sm[wl] & bit) && !(atomicOr(&sm[wl], bit) & bit)) {
            const uint32_t win = vl >> wlog;
            const uint32_t at = atomicAdd(&s.own_cnt[win], 1u);
            stage[(win << wlog) + at] = make_uint2(vl & wmask, uu[k]);
          }
        }
      }
    }
    __syncthreads();
  }
  OWN_MARK(3);
#if GK_OWN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 290) {
    P.ctrl->ts[100 + blockIdx.x] = globaltimer();
    P.ctrl->tag[100 + blockIdx.x] = 'g';
  }
#endif
  for (int i = threadIdx.x; i < nw; i += kBlock) atomicOr(nextbm + w0 + i, sm[i]);
  __syncthreads();
  OWN_MARK(4);
  // Parents, window by window: gather the window's logged claims into
  // shared memory (the slice's space), then store them in vertex order
  // (coalesced: measured faster than storing the log entries directly).
  // The next window's log entries are loaded while this window is written
  // back (kOwnPf per thread in registers, the rest of a full window read
  // directly): the log's DRAM round trip leaves the per-window critical path.
  int32_t* par = reinterpret_cast<int32_t*>(sm);
  const long long id0 = w0 * 32;
  const int ws = 1 << wlog;
  constexpr int kOwnPf = 4;
  auto next_win = [&](int w) {
    while (w < nwin && s.own_cnt[w] == 0) w++;  // uniform
    return w;
  };
  uint2 pf[kOwnPf];
  auto fetch = [&](int w) {
    const unsigned cnt = w < nwin ? s.own_cnt[w] : 0u;
    const uint2* st = stage + ((int64_t)w << wlog);
#pragma unroll
    for (int k = 0; k < kOwnPf; k++) {
      const unsigned j = threadIdx.x + k * kBlock;
      pf[k] = j < cnt ? __ldcg(st + j) : make_uint2(0xffffffffu, 0u);
    }
  };
  int win = next_win(0);
  fetch(win);
  for (int i = threadIdx.x; i < ws; i += kBlock) par[i] = -2;
  __syncthreads();
  while (win < nwin) {
    const unsigned cnt = s.own_cnt[win];
    const long long lo = id0 + ((long long)win << wlog);
#pragma unroll
    for (int k = 0; k < kOwnPf; k++)
      if (pf[k].x != 0xffffffffu) par[pf[k].x] = (int32_t)pf[k].y;
    const uint2* st = stage + ((int64_t)win << wlog);
    for (unsigned j = threadIdx.x + kOwnPf * kBlock; j < cnt; j += kBlock) {
      const uint2 c = __ldcg(st + j);
      par[c.x] = (int32_t)c.y;
    }
    const int nwin2 = next_win(win + 1);
    fetch(nwin2);
    __syncthreads();
    for (int i = threadIdx.x; i < ws; i += kBlock) {
      const int32_t pv = par[i];
      if (pv != -2) {
        *parent_slot(P, (uint32_t)(lo + i)) = pv;
        par[i] = -2;
      }
    }
    __syncthreads();
    win = nwin2;
  }
  OWN_MARK(5);
  if (blockIdx.x == 0 && threadIdx.x == 0 && GK_OWN_TRACE) {
    P.ctrl->ts[410] = nown;
    P.ctrl->ts[411] = (unsigned long long)nwin;
    P.ctrl->tag[410] = P.ctrl->tag[411] = 'n';
  }
}

// Sum of max(deg, 1) over the claimed vertices of 32 consecutive bitmap
// words (lane l: word w0 + l, claim bits cl) -- bfs.hpp:83's -old with
// bfs.hpp:130's encoding.  The claims are numbered by a warp scan and spread
// over the lanes, 4 per lane in flight; claim c's word is found by a
// shuffle search of the scan, so the offset reads go out in vertex order.
// Every lane of the warp must call it; returns this lane's part.
__device__ __forceinline__ long long claim_degrees(const BfsParams& P, long long w0, uint32_t cl) {
  const unsigned lane = lane_id();
  long long scout = 0;
  if (!__ballot_sync(kFull, cl != 0u)) return 0;
  const int cnt = __popc(cl);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, o);
    if ((int)lane >= o) incl += y;
  }
  const int excl = incl - cnt;
  const int total = __shfl_sync(kFull, incl, 31);
  for (int c0 = 0; c0 < total; c0 += 128) {
    int64_t o0[4], o1[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int c = c0 + 32 * k + (int)lane;
      int lo = 0;  // last lane whose first claim is <= c
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int e = __shfl_sync(kFull, excl, lo + step);
        if (e <= c) lo += step;
      }
      const uint32_t m = __shfl_sync(kFull, cl, lo);
      const int ex = __shfl_sync(kFull, excl, lo);
      o0[k] = o1[k] = -1;
      if (c < total) {
        const int64_t v = (w0 + lo) * 32 + (int64_t)__fns(m, 0, c - ex + 1);
        o0[k] = offv(P, P.out_off, v);
        o1[k] = offv(P, P.out_off, v + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int64_t d = o1[k] - o0[k];
      if (o0[k] >= 0) scout += d ? d : 1;
    }
  }
  return scout;
}

// ---- degrees of the vertices a large top-down step claimed ----------------
// scout = sum of -old over the claims (bfs.hpp:83) = sum of max(deg, 1)
// with the degree encoding, or the claim count without it (bfs.hpp:129).
// A warp walks 32 bitmap words (1024 vertices) per iteration in vertex
// order: lane l owns word l (claims = next & ~visited become the next
// frontier and are folded into visited), then the claimed vertices are
// numbered by a warp prefix sum and spread over the lanes, four per lane in
// flight, so the offset reads are sorted, mostly coalesced runs.  The next
// iteration's words are loaded one iteration ahead.
__device__ void td_scout_bits(const BfsParams& P, uint32_t* bm, int lvl, bool encode,
                              long long& scout, long long& count) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  auto load2 = [&](long long w0, uint32_t& nx, uint32_t& vis) {
    const long long w = w0 + lane;
    nx = vis = 0u;
    if (w < P.w32) {
      nx = ld_bits(bm + w);
      vis = ld_bits(P.visited + w);
    }
  };
  long long w0 = gw * 32;
  uint32_t nx, vis;
  load2(w0, nx, vis);
  for (; w0 < P.w32; w0 += nw * 32) {
    uint32_t nx_n, vis_n;
    load2(w0 + nw * 32, nx_n, vis_n);
    const uint32_t cl = nx & ~vis;
    if (w0 + lane < P.w32) {
      if (cl != nx) bm[w0 + lane] = cl;
      if (cl) P.visited[w0 + lane] = vis | cl;
    }
    count += __popc(cl);
    if (!encode) {
      scout += __popc(cl);
    } else {
      scout += claim_degrees(P, w0, cl);
    }
    if (cl) {
      if (P.want_depth)
        for (uint32_t m = cl; m; m &= m - 1) P.depth[(w0 + lane) * 32 + (__ffs(m) - 1)] = lvl + 1;
    }
    nx = nx_n;
    vis = vis_n;
  }
}

// ---- bottom-up sweep (bfs.hpp:47-66) ---------------------------------------
// A warp takes a task of 32 consecutive bitmap words (1024 vertices): lane l
// loads word l and the task's pending vertices (not visited; visited starts
// as the graph's dead set, so vertices without in-edges never appear) are
// numbered by a warp prefix sum and listed once in shared memory.  Every
// lane keeps kBuSlots vertices in flight.  A slot is refilled with the next
// pending vertex as soon as its vertex resolves: the refill issues the loads
// of the vertex's two in-offsets and the slot starts its rounds in the next
// loop iteration, so that latency overlaps the other slots' rounds.  Per
// round a slot tests the next kPerRound in-neighbours (the first alone, then
// the rest together).  After kLaneRounds rounds a still-unresolved vertex is
// deferred to the long list, scanned after the sweep by whole warps with a
// ballot per 32 neighbours.  The chosen parent is the first in-neighbour
// (ascending) whose front bit is set, as in bfs.hpp:55-60.  Results are
// OR-ed into per-warp shared-memory words and written back once per task.
#ifndef GK_BU_SLOTS
#define GK_BU_SLOTS 3  // 2: -0.5%, 4: spills (-8%) on kron27
#endif
constexpr int kBuSlots = GK_BU_SLOTS;
#ifndef GK_BU_PREFETCH_OFF
#define GK_BU_PREFETCH_OFF 0
#endif
constexpr int kBuListWords = 512;  // per warp: 1024 uint16 pending ids
constexpr size_t kBuListBytes = (size_t)kWarps * kBuListWords * 4;
#ifndef GK_BU_PER_ROUND
#define GK_BU_PER_ROUND 4
#endif
constexpr int kPerRound = GK_BU_PER_ROUND;  // in-neighbours tested per slot per round
constexpr int kLaneRounds = 48 / GK_BU_PER_ROUND;  // rounds before a list is deferred to the long list
constexpr int kLaneScan = kPerRound * kLaneRounds;  // in-neighbours a lane tests (4-entry rounds)
constexpr int kSparseScan = kLaneScan;  // entries sp_scan tests before deferring a list to bu_long

// Where bu_long resumes a list bu_step deferred.
__device__ __forceinline__ int64_t bu_resume(int64_t o) { return o + kLaneScan; }

template <bool kSmem>
__device__ __forceinline__ bool front_bit(const uint32_t* front, uint32_t u) {
  const uint32_t w = kSmem ? front[u >> 5] : ld_front(front + (u >> 5));
  return (w >> (u & 31u)) & 1u;
}

template <bool kSmem>
__device__ void bu_step(const BfsParams& P, SmemT& s, unsigned ph, const uint32_t* front, uint32_t* next,
                        int lvl, unsigned long long long_base, int tw_log, long long& awake, uint32_t* wsm) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  // kList (front read from global memory, so the dynamic shared memory is
  // free): the task's pending vertices are listed once in shared memory and
  // a refill is one list read instead of a shuffle binary search.
  constexpr bool kList = !kSmem;
  uint16_t* lst = nullptr;
  if constexpr (kList) lst = reinterpret_cast<uint16_t*>(wsm + warp * kBuListWords);
  uint32_t* acc_n = s.bu_acc[warp];
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  // A task is 2^tw_log consecutive words (<= 32): small graphs use small
  // tasks so every warp gets work.
  const int tw = 1 << tw_log;
  const long long ntasks = (P.w_hi - P.w_lo + tw - 1) >> tw_log;  // over the owned words
  // First task static, later ones claimed dynamically (per-task work varies
  // with the pending density and list lengths); the next claim is issued
  // when a task starts, so its round trip hides behind the task.
  unsigned long long* tctr = &rset(P, ph)[kTile];
  for (long long t = gw; t < ntasks;) {
    long long tnext = 0;
    if (lane == 0) tnext = nw + (long long)atomicAdd(tctr, 1ull);
    const long long tbase = P.w_lo + (t << tw_log);
    const long long w = tbase + lane;
    uint32_t vis = 0xffffffffu, pad = 0u;
    if ((int)lane < tw && w < P.w_hi) {
      vis = ld_bits(P.visited + w);
      const int64_t rem = P.n - w * 32;  // mask off ids >= n in the last word
      if (rem < 32) pad = 0xffffffffu << rem;
    }
    const uint32_t pm = ~(vis | pad);
    const int cnt = __popc(pm);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(kFull, incl, 31);
    if constexpr (kList) {
      uint32_t m = pm;
      int pos = excl;
#if GK_BU_PREFETCH_OFF
      uint32_t last_sec = 0xffffffffu;
#endif
      while (m) {
        const int bt = __ffs(m) - 1;
        m &= m - 1;
        lst[pos++] = (uint16_t)((lane << 5) | bt);
#if GK_BU_PREFETCH_OFF
        const uint32_t sec = (uint32_t)bt >> 2;  // 4 offsets per 32-byte sector
        if (sec != last_sec) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.in_off + w * 32 + bt));
          last_sec = sec;
        }
#endif
      }
    }
    acc_n[lane] = 0u;
    __syncwarp();
    int next_c = 0;
    uint32_t v[kBuSlots], d[kBuSlots], rounds[kBuSlots];
    int64_t b[kBuSlots], e[kBuSlots];
    int st[kBuSlots];  // 0 empty, 1 offsets in flight, 2 in-list rounds
#pragma unroll
    for (int k = 0; k < kBuSlots; k++) {
      st[k] = 0;
      v[k] = d[k] = rounds[k] = 0;
      b[k] = e[k] = 0;
    }
    for (;;) {
      // refill empty slots with the next pending vertices of the task
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        const bool need = st[k] == 0;
        const unsigned nm = __ballot_sync(kFull, need);
        if (nm == 0 || next_c >= total) continue;  // uniform: nothing to hand out
        const int c = next_c + __popc(nm & lanemask_lt());
        next_c += __popc(nm);
        if constexpr (kList) {
          if (need && c < total) {
            const uint32_t en = lst[c];
            v[k] = (uint32_t)((tbase + (en >> 5)) * 32 + (en & 31u));
            b[k] = offv(P, P.in_off, v[k]);
            e[k] = offv(P, P.in_off, v[k] + 1);
            st[k] = 1;
          }
          continue;
        }
        int lo = 0;  // word holding the c-th pending vertex: last lane with excl <= c
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int ex = __shfl_sync(kFull, excl, lo + step);
          if (ex <= c) lo += step;
        }
        const uint32_t m = __shfl_sync(kFull, pm, lo);
        const int ex = __shfl_sync(kFull, excl, lo);
        if (need && c < total) {
          v[k] = (uint32_t)((tbase + lo) * 32 + (int)__fns(m, 0, c - ex + 1));
          b[k] = offv(P, P.in_off, v[k]);
          e[k] = offv(P, P.in_off, v[k] + 1);
          st[k] = 1;
        }
      }
      bool active = false;
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) active |= st[k] != 0;
      if (__ballot_sync(kFull, active) == 0) {
        if (next_c >= total) break;
        continue;
      }
      uint32_t u[kBuSlots][kPerRound];
#pragma unroll
      for (int k = 0; k < kBuSlots; k++)
#pragma unroll
        for (int j = 0; j < kPerRound; j++)
          u[k][j] = (st[k] == 2 && d[k] > (uint32_t)j) ? ld_nb(P.in_nb + b[k] + j) : kNoVertex;
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        if (st[k] != 2) continue;
        bool hit = false;
        uint32_t par = 0;
        // The first in-neighbour's front bit alone, then the rest of the
        // round's at once: one lookup when the first hits, two latencies
        // instead of up to kPerRound otherwise.
        uint32_t fw[kPerRound];
        fw[0] = u[k][0] != kNoVertex ? (kSmem ? front[u[k][0] >> 5] : ld_front(front + (u[k][0] >> 5))) : 0u;
        if ((fw[0] >> (u[k][0] & 31u)) & 1u) {
          hit = true;
          par = u[k][0];
        } else {
#pragma unroll
          for (int j = 1; j < kPerRound; j++)
            fw[j] = u[k][j] != kNoVertex ? (kSmem ? front[u[k][j] >> 5] : ld_front(front + (u[k][j] >> 5))) : 0u;
#pragma unroll
          for (int j = 1; j < kPerRound; j++)
            if (!hit && ((fw[j] >> (u[k][j] & 31u)) & 1u)) {
              hit = true;
              par = u[k][j];
            }
        }
        if (hit) {
#ifndef GK_BU_NO_PARENT  // diagnostic A/B only (results invalid without it)
          P.parent[v[k]] = (int32_t)par;
#endif
          if (P.want_depth) P.depth[v[k]] = lvl + 1;
          atomicOr(&acc_n[(v[k] >> 5) - tbase], 1u << (v[k] & 31u));
          st[k] = 0;
        } else {
          const uint32_t tk = d[k] < (uint32_t)kPerRound ? d[k] : (uint32_t)kPerRound;
          b[k] += tk;
          d[k] -= tk;
          if (d[k] == 0) {
            st[k] = 0;  // exhausted: not reached at this level
          } else if (++rounds[k] >= kLaneRounds) {
            P.queue[long_base + atomicAdd(&rset(P, ph)[kLongCount], 1ull)] = v[k];
            if (GK_SHARDED_STEPS) atomicAdd(&P.ctrl->cnt[ph & 3][kWork], 1ull);
            st[k] = 0;
          }
        }
      }
      // slots refilled this iteration start their rounds in the next one
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        if (st[k] == 1) {
          d[k] = (uint32_t)(e[k] - b[k]);  // < 2^32 (in-degree of one vertex)
          rounds[k] = 0;
          st[k] = d[k] ? 2 : 0;
        }
      }
    }
    __syncwarp();
    if ((int)lane < tw && w < P.w_hi) {
      const uint32_t nbits = acc_n[lane];
      next[w] = nbits;
      if (nbits) P.visited[w] = vis | nbits;
      awake += __popc(nbits);
    }
    __syncwarp();
    t = __shfl_sync(kFull, tnext, 0);
  }
}

// Long in-lists deferred by bu_step: one warp per vertex, ballot over 32
// neighbours at a time, resuming after the kLaneScan in-neighbours bu_step
// tested.
template <bool kSmem, bool kPull = false, bool kSparse = false>
__device__ void bu_long(const BfsParams& P, const uint32_t* front, uint32_t* next, const uint32_t* lst,
                        unsigned long long count, int lvl, long long& awake, long long& scout) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  for (long long i = gw; i < (long long)count; i += nw) {
    const uint32_t v = __ldcg(lst + i);
    const int64_t le = offv(P, P.in_off, v + 1);
    const int64_t lb = offv(P, P.in_off, v);
    for (int64_t j = kSparse ? lb + kSparseScan : bu_resume(lb); j < le; j += 32) {
      const int64_t jj = j + lane;
      bool h = false;
      uint32_t u = 0;
      if (jj < le) {
        u = ld_nb(P.in_nb + jj);
        h = front_bit<kSmem>(front, u);
      }
      const unsigned bal = __ballot_sync(kFull, h);
      if (bal) {
        const uint32_t hu = __shfl_sync(kFull, u, __ffs(bal) - 1);
        if (lane == 0) {
          P.parent[v] = (int32_t)hu;
          if (P.want_depth) P.depth[v] = lvl + 1;
          atomicOr(next + (v >> 5), 1u << (v & 31u));
          atomicOr(P.visited + (v >> 5), 1u << (v & 31u));
          awake++;
          if constexpr (kPull) {  // top-down result of the claim (bfs.hpp:83)
            const int64_t dg = offv(P, P.out_off, v + 1) - offv(P, P.out_off, v);
            scout += dg ? dg : 1;
          }
        }
        break;
      }
    }
  }
}

// ---- sparse sweeps: few vertices left unreached ----------------------------
// Once the unreached (pending) vertices are few, a bottom-up step -- or a
// top-down step of the reference's schedule whose frontier is larger than
// the pending set, executed as a pull (same claimed set: unvisited vertices
// with an in-neighbour in the frontier; parents are any frontier
// in-neighbour, as top-down's racy claims also are) -- costs one list pass:
// sp_list writes the pending vertices to a list (and clears next),
// sp_scan gives each one a thread that scans its in-list in ascending order
// (first hit = parent, as bfs.hpp:55-60) for up to kSparseScan entries and
// defers longer lists to bu_long.  A full bu_step sweep costs ~0.1 ms at
// scale 27 even when nothing is pending (one dependent chain per task).

__device__ void sp_list(const BfsParams& P, unsigned long long* ctr, uint32_t* lst, uint32_t* next) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  for (long long seg = P.w_lo + gw * 256; seg < P.w_hi; seg += nw * 256) {
    const long long w0 = seg + lane * 8;
    uint32_t wd[8];
    if (w0 + 8 <= P.w_hi && (w0 + 8) * 32 <= P.n) {  // two 16-byte loads and stores
      const uint4 x = __ldcg(reinterpret_cast<const uint4*>(P.visited + w0));
      const uint4 y = __ldcg(reinterpret_cast<const uint4*>(P.visited + w0 + 4));
      wd[0] = ~x.x; wd[1] = ~x.y; wd[2] = ~x.z; wd[3] = ~x.w;
      wd[4] = ~y.x; wd[5] = ~y.y; wd[6] = ~y.z; wd[7] = ~y.w;
      reinterpret_cast<uint4*>(next + w0)[0] = make_uint4(0u, 0u, 0u, 0u);
      reinterpret_cast<uint4*>(next + w0)[1] = make_uint4(0u, 0u, 0u, 0u);
    } else {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const long long w = w0 + j;
        wd[j] = 0u;
        if (w < P.w_hi) {
          const int64_t rem = P.n - w * 32;
          const uint32_t pad = rem < 32 ? 0xffffffffu << rem : 0u;
          wd[j] = ~(ld_bits(P.visited + w) | pad);  // visited includes the dead set
          next[w] = 0u;
        }
      }
    }
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) cnt += __popc(wd[j]);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    if (total == 0) continue;  // uniform
    unsigned long long q = 0;
    if (lane == 0) q = atomicAdd(ctr, (unsigned long long)total);
    q = __shfl_sync(kFull, q, 0) + (incl - cnt);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      for (uint32_t m = wd[j]; m; m &= m - 1) lst[q++] = (uint32_t)((w0 + j) * 32 + (__ffs(m) - 1));
    }
  }
}

template <bool kPull>
__device__ void sp_scan(const BfsParams& P, unsigned ph, const uint32_t* front, uint32_t* next, const uint32_t* lst,
                        unsigned long long cnt, uint32_t* lng, int lvl, long long& found, long long& scout) {
  // two list entries per thread in flight, their in-list rounds interleaved
  constexpr int kS = 2;
  const long long gtid = (long long)cta_id(P) * kBlock + threadIdx.x;
  const long long gthreads = (long long)cta_count(P) * kBlock;
  for (long long i0 = gtid; i0 < (long long)cnt; i0 += kS * gthreads) {
    uint32_t v[kS], par[kS];
    int64_t o0[kS], o1[kS], j[kS], lim[kS];
    bool act[kS], hit[kS];
#pragma unroll
    for (int k = 0; k < kS; k++) {
      const long long i = i0 + k * gthreads;
      act[k] = i < (long long)cnt;
      hit[k] = false;
      par[k] = 0;
      v[k] = act[k] ? __ldcg(lst + i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kS; k++) {
      o0[k] = act[k] ? offv(P, P.in_off, v[k]) : 0;
      o1[k] = act[k] ? offv(P, P.in_off, v[k] + 1) : 0;
      lim[k] = o1[k] - o0[k] > kSparseScan ? o0[k] + kSparseScan : o1[k];
      j[k] = o0[k];
      act[k] = act[k] && j[k] < lim[k];
    }
    while (act[0] || act[1]) {
      uint32_t u[kS][kPerRound], fw[kS][kPerRound];
#pragma unroll
      for (int k = 0; k < kS; k++)
#pragma unroll
        for (int q = 0; q < kPerRound; q++) u[k][q] = act[k] && j[k] + q < lim[k] ? ld_nb(P.in_nb + j[k] + q) : kNoVertex;
#pragma unroll
      for (int k = 0; k < kS; k++)
#pragma unroll
        for (int q = 0; q < kPerRound; q++) fw[k][q] = u[k][q] != kNoVertex ? ld_front(front + (u[k][q] >> 5)) : 0u;
#pragma unroll
      for (int k = 0; k < kS; k++) {
#pragma unroll
        for (int q = 0; q < kPerRound; q++)
          if (!hit[k] && ((fw[k][q] >> (u[k][q] & 31u)) & 1u)) {
            hit[k] = true;
            par[k] = u[k][q];
          }
        j[k] += kPerRound;
        act[k] = act[k] && !hit[k] && j[k] < lim[k];
      }
    }
#pragma unroll
    for (int k = 0; k < kS; k++) {
      if (hit[k]) {
        const uint32_t vv = v[k];
        P.parent[vv] = (int32_t)par[k];
        if (P.want_depth) P.depth[vv] = lvl + 1;
        atomicOr(next + (vv >> 5), 1u << (vv & 31u));
        atomicOr(P.visited + (vv >> 5), 1u << (vv & 31u));
        found++;
        if constexpr (kPull) {
          const int64_t dg = offv(P, P.out_off, vv + 1) - offv(P, P.out_off, vv);
          scout += dg ? dg : 1;
        }
      } else if (i0 + k * gthreads < (long long)cnt && o1[k] - o0[k] > kSparseScan) {
        lng[atomicAdd(&rset(P, ph)[kLongCount], 1ull)] = v[k];
      }
    }
  }
}

// One sparse step: list, scan, long lists.  found / scout (kPull) are the
// grid totals (uniform) when it returns true.
template <bool kPull>
__device__ bool sparse_step(const BfsParams& P, SmemT& s, unsigned& ph, const uint32_t* front, uint32_t* next,
                            int lvl, long long& found, long long& scout) {
  uint32_t* lst = reinterpret_cast<uint32_t*>(P.chunks);  // free outside top-down steps
  sp_list(P, &rset(P, ph)[kAppend], lst, next);
  if (!grid_sync(P, s, ph, kTagZero)) return false;
  const unsigned long long cnt = s.snap[kAppend];
  long long f = 0, sc = 0;
  sp_scan<kPull>(P, ph, front, next, lst, cnt, lst + cnt, lvl, f, sc);
  unsigned set = ph & 3;
  block_add(f, &P.ctrl->cnt[set][kSum], s);
  if (kPull) block_add(sc, &P.ctrl->cnt[set][kCount], s);
  if (!grid_sync(P, s, ph, kPull ? kTagPull : kTagBU)) return false;
  found = (long long)s.snap[kSum];
  scout = kPull ? (long long)s.snap[kCount] : 0;
  const unsigned long long nlong = s.snap[kLongCount];
  if (nlong) {
    f = sc = 0;
    bu_long<false, kPull, true>(P, front, next, lst + cnt, nlong, lvl, f, sc);
    set = ph & 3;
    block_add(f, &P.ctrl->cnt[set][kSum], s);
    if (kPull) block_add(sc, &P.ctrl->cnt[set][kCount], s);
    if (!grid_sync(P, s, ph, kTagLong)) return false;
    found += (long long)s.snap[kSum];
    if (kPull) scout += (long long)s.snap[kCount];
  }
  return true;
}

// ---- BitmapToQueue (bfs.hpp:99-113) ----------------------------------------
__device__ void b2q(const BfsParams& P, const QApp& qa, const uint32_t* front) {
  // A warp takes 256 words (lane l: 8 consecutive words, two 16-byte
  // loads), numbers their vertices with a warp scan and appends them with
  // one fetch-add: no CTA barriers, and few enough counter atomics that a
  // sparse front costs about one pass over the bitmap.
  const unsigned lane = lane_id();
  const long long gw = ((long long)cta_id(P) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(P) * kBlock) >> 5;
  for (long long seg = P.w_lo + gw * 256; seg < P.w_hi; seg += nw * 256) {
    const long long w0 = seg + lane * 8;
    uint32_t wd[8];
    if (w0 + 8 <= P.w_hi) {
      const uint4 x = __ldcg(reinterpret_cast<const uint4*>(front + w0));
      const uint4 y = __ldcg(reinterpret_cast<const uint4*>(front + w0 + 4));
      wd[0] = x.x; wd[1] = x.y; wd[2] = x.z; wd[3] = x.w;
      wd[4] = y.x; wd[5] = y.y; wd[6] = y.z; wd[7] = y.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; j++) wd[j] = w0 + j < P.w_hi ? __ldcg(front + w0 + j) : 0u;
    }
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) cnt += __popc(wd[j]);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    if (total == 0) continue;  // uniform
    unsigned long long q = 0;
    if (lane == 0) q = qa.base + atomicAdd(qa.ctr, (unsigned long long)total);
    q = __shfl_sync(kFull, q, 0) + (incl - cnt);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      for (uint32_t m = wd[j]; m; m &= m - 1) P.queue[q++] = (uint32_t)((w0 + j) * 32 + (__ffs(m) - 1));
    }
  }
}

// exec: how the step ran when not as its direction names (0; 'P' a
// bottom-up step executed as a push, 'U' a top-down step executed as a pull)
__device__ void log_step(const BfsParams& P, long long idx, int dir, long long frontier,
                         long long result, long long etc, int exec = 0) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && idx < P.step_cap) {
    gk_step st;
    st.dir = dir;
    st.pad = exec;
    st.frontier = frontier;
    st.result = result;
    st.edges_to_check = etc;
    P.steps[idx] = st;
  }
}

}  // namespace
}  // namespace gk
