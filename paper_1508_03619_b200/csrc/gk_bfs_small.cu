// gk_bfs_small.cu -- the whole traversal of a small graph inside ONE
// thread-block cluster (config 1 regime: n <= 8192 x cluster CTAs, every
// bitmap resident in shared memory).
//
// On a graph this small the grid kernel (bfs_persistent) pays a 296-CTA grid
// barrier and several dependent L2 round trips per phase, 4-6 phases per
// level: ~80 us per kron16 BFS for ~2 MB of traffic.  Here the cluster's CTAs
// (16, or 8 if the device will not co-schedule 16) each hold a full copy of
// the visited and frontier bitmaps in shared memory and own a slice of the
// vertex ids (CTA c: bitmap words [c*Wc, (c+1)*Wc)).  One level is:
//   top-down (bfs.hpp:68-91), by the frontier's size:
//     * <= kSmRedE edges: every CTA expands the whole frontier against its
//       own (identical) visited copy -- the same claimed set everywhere, the
//       owner of a vertex stores its parent; no barrier, no DSMEM;
//     * <= kSmWon vertices: every CTA holds the whole frontier list (the
//       won lists of the last level, gathered with its slices) and takes
//       1/C of the edges; a claim goes to the owner's slice as one DSMEM
//       atomicOr and the single winner stores the parent, keeps the degree
//       it read with the claim (-old of bfs.hpp:83, or deg for
//       kTopDownRescan, bfs.hpp:161-167) and lists the vertex;
//     * larger: each CTA expands its own slice, claims in a local bitmap
//       (racing claimers store valid parents, as on the CPU), and after a
//       barrier the owners OR the C copies over DSMEM and sum the degrees;
//   bottom-up (bfs.hpp:47-66): each CTA scans its own pending vertices'
//     in-lists in ascending order against the replicated front -- the first
//     hit is the parent, exactly the reference's choice;
//   then: each CTA pushes its counters into every CTA (DSMEM stores), one
//     cluster barrier, and every CTA gathers the C new slices (and the won
//     lists, when a small top-down level follows) into its own copies and
//     sums the counters, so every CTA takes the same alpha/beta decision
//     (bfs.hpp:139-169).
// The step log, counters and results are the grid kernel's; the trial is one
// CUDA graph launch (pool allocation node + this kernel; it initialises the
// control block, the parent array and its bitmaps itself).
#include <cooperative_groups.h>

#include "gk_persistent.cuh"

namespace gk {
namespace {

namespace cg = cooperative_groups;

#ifndef GK_SM_BLOCK
#define GK_SM_BLOCK 512  // kron16: 1024 threads -15%, 256 -5%
#endif
constexpr int kSmBlock = GK_SM_BLOCK;
constexpr int kSmWarps = kSmBlock / 32;
constexpr int kSmMaxW = 4096;  // bitmap words: n <= 2^17
constexpr int kSmCap = 8192;   // list entries per CTA (>= one CTA's slice of ids)
constexpr int kSmSlice = kSmCap / 32;  // owned bitmap words per CTA, at most
constexpr int kSmWon = 2048;   // won-list entries per CTA (more: the next level lists from the bitmap)
constexpr int kSmRounds = 4;
#ifndef GK_SM_REDE
#define GK_SM_REDE 4096
#endif
// Top-down levels expanding at most this many edges run redundantly in
// every CTA (no cluster barrier, no DSMEM); <= kSmCap, so the new frontier
// list always fits.
constexpr int kSmRedE = GK_SM_REDE;
static_assert(kSmRedE <= kSmCap && kSmRedE <= kSmMaxW, "a redundant level's new frontier must fit the lists");
#ifndef GK_SM_BUW
#define GK_SM_BUW 2  // slots x in-neighbours per round: 2 x 8 (kron16 +2% over 4 x 4; 16 x 1, 3 x 8 equal, 2 x 16 -1%)
#endif
#ifndef GK_SM_TDW
#define GK_SM_TDW 4
#endif
constexpr int kSmBuW = GK_SM_BUW;  // bottom-up: pending vertices per thread in flight
#ifndef GK_SM_BUR
#define GK_SM_BUR 8
#endif
constexpr int kSmBuR = GK_SM_BUR;  // bottom-up: in-neighbours per vertex per round
constexpr int kSmTdW = GK_SM_TDW;  // top-down: edges per thread in flight   // bottom-up: 4-neighbour rounds per thread before the warp takes a list

struct __align__(16) SmShared {
  uint32_t vis[kSmMaxW];          // visited (replicated; starts as the dead set)
  uint32_t front[kSmMaxW];        // current frontier (replicated)
  uint32_t nxt[kSmMaxW];          // top-down: this CTA's claims (all ids)
  uint32_t slice[3][kSmSlice];    // this CTA's slice of level L's new frontier in [L % 3]
  uint32_t ids[kSmCap];           // listed vertices (frontier / pending)
  uint32_t pre[kSmCap + 1];       // top-down: exclusive degree prefix; bottom-up: long list
  uint32_t off[kSmCap];           // top-down: out_off of the listed vertex (m < 2^32)
  uint4 wl[2][kSmWon];            // won lists by level parity: {vertex, out_off, out-degree, 0} of the
                                  // vertices this CTA added to the frontier in a top-down level
  uint4 cin[3][16];               // level L in [L % 3], pushed by CTA r into every CTA's [r]:
                                  // {new vertices, degree total, no won list, won-list length}
  uint4 red4[2][kSmWarps];        // per-warp partial sums, two alternating slots
  unsigned nlong;
  unsigned nwon;
  unsigned nred;  // redundant level: vertices claimed so far (listed in front)
};

// Block-wide exclusive scan / sums of 32-bit values with ONE barrier: warp
// scans (shuffles) or REDUX sums, per-warp totals in smem slot rs (the two
// slots alternate, so a slot is rewritten only after every thread passed
// the barrier of the call in between), every thread sums the totals it needs.
__device__ __forceinline__ unsigned sm_exscan(unsigned x, unsigned* total, SmShared& S, int& rs) {
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o);
    if ((int)lane >= o) incl += y;
  }
  uint4* r = S.red4[rs];
  if (lane == 31) r[warp].x = incl;
  rs ^= 1;
  __syncthreads();
  unsigned base = 0, tot = 0;
#pragma unroll 8
  for (int i = 0; i < kSmWarps; i++) {
    const unsigned v = r[i].x;
    base += (unsigned)i < warp ? v : 0u;
    tot += v;
  }
  *total = tot;
  return base + incl - x;
}

__device__ __forceinline__ uint3 sm_sum3(unsigned a, unsigned b, unsigned c, SmShared& S, int& rs) {
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  a = __reduce_add_sync(kFull, a);
  b = __reduce_add_sync(kFull, b);
  c = __reduce_add_sync(kFull, c);
  uint4* r = S.red4[rs];
  if (lane == 0) r[warp] = make_uint4(a, b, c, 0u);
  rs ^= 1;
  __syncthreads();
  uint3 t = make_uint3(0u, 0u, 0u);
#pragma unroll 8
  for (int i = 0; i < kSmWarps; i++) {
    const uint4 v = r[i];
    t.x += v.x;
    t.y += v.y;
    t.z += v.z;
  }
  return t;
}

// List the set bits of words [wa, wb) of bm (complemented when kNot) into
// S.ids in ascending id order; returns the count (uniform).
template <bool kNot>
__device__ int sm_list(SmShared& S, const uint32_t* bm, int wa, int wb, int& rs) {
  const int nw = wb - wa;
  const int q = (nw + kSmBlock - 1) / kSmBlock;
  const int j0 = wa + (int)threadIdx.x * q, j1 = min(wb, j0 + q);
  unsigned cnt = 0;
  for (int j = j0; j < j1; j++) cnt += __popc(kNot ? ~bm[j] : bm[j]);
  unsigned total;
  int pos = (int)sm_exscan(cnt, &total, S, rs);
  for (int j = j0; j < j1; j++) {
    uint32_t w = kNot ? ~bm[j] : bm[j];
    while (w) {
      const int b = __ffs(w) - 1;
      w &= w - 1;
      S.ids[pos++] = (uint32_t)(j * 32 + b);
    }
  }
  __syncthreads();
  return (int)total;
}

// Level end, before the cluster barrier: this CTA's counters into every
// CTA's cin[q][c] (DSMEM stores; the barrier's release / acquire orders
// them), so after the barrier every CTA sums them locally.
__device__ __forceinline__ void sm_push(SmShared& S, cg::cluster_group& cl, int C, int c, int q, uint4 v) {
  if ((int)threadIdx.x < C) *cl.map_shared_rank(&S.cin[q][c], (int)threadIdx.x) = v;
}

struct SmTot {
  long long cnt, sc;
  bool lists;  // every CTA's won list holds its share of the new frontier
};
__device__ __forceinline__ SmTot sm_totals(const SmShared& S, int C, int q) {
  SmTot r{0, 0, true};
  for (int k = 0; k < C; k++) {
    const uint4 v = S.cin[q][k];
    r.cnt += v.x;
    r.sc += v.y;
    r.lists &= v.z == 0u;
  }
  return r;
}

// After the level's cluster barrier: gather the C new slices of level
// buffer q into front / visited (16-byte DSMEM loads; Wc is a multiple of
// 4 and slice words past a CTA's range stay zero), clear the local claims,
// and -- when the next level is a top-down one over the won lists (wl
// buffer rp, k entries) -- gather the lists too, in the same round trip:
// thread t takes entries [4t, 4t+4), so one scan gives the degree prefix.
__device__ void sm_gather(SmShared& S, cg::cluster_group& cl, int C, int W, int Wc, int q, bool with_list, int rp,
                          int k, int& rs) {
  const int t = threadIdx.x;
  constexpr int kPerL = kSmWon / kSmBlock;
  uint4 sl[kSmMaxW / 4 / kSmBlock];
#pragma unroll
  for (int i = 0; i < kSmMaxW / 4 / kSmBlock; i++) {
    const int j = 4 * (t + i * kSmBlock);
    sl[i] = make_uint4(0u, 0u, 0u, 0u);
    if (j < W) {
      const int r = j / Wc;
      sl[i] = *reinterpret_cast<const uint4*>(cl.map_shared_rank(&S.slice[q][0], r) + (j - r * Wc));
    }
  }
  uint4 le[kPerL];
  if (with_list) {
    int pre[17];  // exclusive prefix of the C won-list lengths
    pre[0] = 0;
#pragma unroll
    for (int r = 0; r < 16; r++) pre[r + 1] = pre[r] + (r < C ? (int)S.cin[q][r].w : 0);
#pragma unroll
    for (int e = 0; e < kPerL; e++) {
      const int i = t * kPerL + e;
      le[e] = make_uint4(0u, 0u, 0u, 0u);
      if (i < k) {
        int r = 0;
#pragma unroll
        for (int b = 8; b > 0; b >>= 1)
          if (r + b < C && pre[r + b] <= i) r += b;
        le[e] = cl.map_shared_rank(&S.wl[rp][0], r)[i - pre[r]];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kSmMaxW / 4 / kSmBlock; i++) {
    const int j = 4 * (t + i * kSmBlock);
    if (j < W) {
      const uint4 w = sl[i];
      *reinterpret_cast<uint4*>(&S.front[j]) = w;
      uint4 v = *reinterpret_cast<const uint4*>(&S.vis[j]);
      v.x |= w.x;
      v.y |= w.y;
      v.z |= w.z;
      v.w |= w.w;
      *reinterpret_cast<uint4*>(&S.vis[j]) = v;
      *reinterpret_cast<uint4*>(&S.nxt[j]) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  if (with_list) {  // ids, offsets and the exclusive degree prefix of the next frontier
    unsigned sum = 0;
#pragma unroll
    for (int e = 0; e < kPerL; e++) sum += le[e].z;
    unsigned tot;
    unsigned x = sm_exscan(sum, &tot, S, rs);
#pragma unroll
    for (int e = 0; e < kPerL; e++) {
      const int i = t * kPerL + e;
      if (i < k) {
        S.ids[i] = le[e].x;
        S.off[i] = le[e].y;
        S.pre[i] = x;
      }
      x += le[e].z;
    }
    if (t == 0) S.pre[k] = tot;
  }
  if (t == 0) S.nwon = 0u;  // the coming level's won list
  __syncthreads();
}

#ifndef GK_SM_TRACE
#define GK_SM_TRACE 0  // diagnostics: CTA 0 logs sub-phase timestamps in the trace instead of one per level
#endif
#if GK_SM_TRACE
#define SM_MARK(ch)                                      \
  do {                                                   \
    if (c == 0 && t == 0 && trace_i + 1 < kTraceCap) {   \
      trace_i++;                                         \
      P.ctrl->ts[trace_i] = clock64();                   \
      P.ctrl->tag[trace_i] = (unsigned char)(ch);        \
    }                                                    \
  } while (0)
#else
#define SM_MARK(ch) \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ bool sm_bit(const uint32_t* bm, uint32_t v) { return (bm[v >> 5] >> (v & 31u)) & 1u; }

__device__ void sm_log(const BfsParams& P, int c, long long idx, int dir, long long frontier, long long result,
                       long long etc) {
  if (c == 0 && threadIdx.x == 0) {
    if (idx < P.step_cap) {
      gk_step st;
      st.dir = dir;
      st.pad = 'S';  // executed by the single-cluster kernel
      st.frontier = frontier;
      st.result = result;
      st.edges_to_check = etc;
      P.steps[idx] = st;
    }
    if (!GK_SM_TRACE && idx + 1 < kTraceCap) {
      P.ctrl->ts[idx + 1] = globaltimer();
      P.ctrl->tag[idx + 1] = (unsigned char)dir;
    }
  }
}

// Back to cluster-wide levels after redundant ones: no CTA still reads an
// earlier level's slices once all reached the first barrier; every slice
// this CTA owns is zeroed; the second barrier orders that before the
// level's claims.
__device__ __forceinline__ void sm_resync(SmShared& S, cg::cluster_group& cl, bool& synced, int wlo, int whi) {
  if (synced) return;
  cl.sync();
  for (int j = threadIdx.x; j < whi - wlo; j += kSmBlock) {
    S.slice[0][j] = 0u;
    S.slice[1][j] = 0u;
    S.slice[2][j] = 0u;
  }
  cl.sync();
  synced = true;
}

// Exclusive prefix of the k list degrees in S.pre (kPer consecutive entries
// per thread), S.pre[k] = total; returns the total.  Ends with a barrier.
__device__ long long sm_prefix(SmShared& S, int k, int& rs) {
  __syncthreads();
  if (k <= kSmBlock) {  // one entry per thread
    const unsigned d = (int)threadIdx.x < k ? S.pre[threadIdx.x] : 0u;
    unsigned tot;
    const unsigned x = sm_exscan(d, &tot, S, rs);
    if ((int)threadIdx.x < k) S.pre[threadIdx.x] = x;
    if (threadIdx.x == 0) S.pre[k] = tot;
    __syncthreads();
    return tot;
  }
  constexpr int kPer = kSmCap / kSmBlock;
  const int i0 = threadIdx.x * kPer;
  uint32_t d[kPer];
  unsigned sum = 0;
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    d[q] = i0 + q < k ? S.pre[i0 + q] : 0u;
    sum += d[q];
  }
  unsigned tot;
  unsigned x = sm_exscan(sum, &tot, S, rs);
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    if (i0 + q < k) S.pre[i0 + q] = (uint32_t)x;
    x += d[q];
  }
  if (threadIdx.x == 0) S.pre[k] = (uint32_t)tot;
  __syncthreads();
  return tot;
}

__global__ void __launch_bounds__(kSmBlock, 1) bfs_small(BfsParams P) {
  extern __shared__ uint4 sm_raw[];
  SmShared& S = *reinterpret_cast<SmShared*>(sm_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), C = (int)cl.num_blocks();
  const int t = threadIdx.x;
  const unsigned lane = t & 31u, warp = t >> 5;
  const int W = (int)P.w32;
  const int Wc = ((W + C - 1) / C + 3) & ~3;  // <= kSmSlice (checked by the host)
  const int wlo = min(W, c * Wc), whi = min(W, wlo + Wc);
  const uint32_t src = P.src;
  const bool encode = P.strategy != GK_BFS_TOP_DOWN_RESCAN;
  int rs = 0;  // reduction slot (sm_exscan / sm_sum3)
#if GK_SM_SPAN  // diagnostics: kernel entry / exit times (globaltimer) in ts[510] / ts[511]
  const unsigned long long t_in = globaltimer();
#endif
#if GK_SM_TRACE
  int trace_i = 0;
  const unsigned long long t_entry = clock64();  // SM cycles in trace mode
#endif

  // ---- init (replaces bfs.hpp:126-138) ----
  if (c == 0) {  // the control block: nothing of it survives from an earlier trial
    uint4* z = reinterpret_cast<uint4*>(P.ctrl);
    for (int i = t; i < (int)(kCtrlClear / 16); i += kSmBlock) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  {
    const long long gt = (long long)c * kSmBlock + t, gn = (long long)C * kSmBlock;
    for (long long i = gt; i < P.n; i += gn) P.parent[i] = -1;
    if (P.want_depth)
      for (long long i = gt; i < P.n; i += gn) P.depth[i] = -1;
  }
  for (int j = t; j < W; j += kSmBlock) {
    S.vis[j] = __ldg(P.dead + j);  // never-reachable vertices and ids >= n start visited
    S.front[j] = 0u;
    S.nxt[j] = 0u;
  }
  for (int j = t; j < 3 * kSmSlice; j += kSmBlock) (&S.slice[0][0])[j] = 0u;
  if (t == 0) {
    S.nwon = 0u;  // the first level's won list (later levels: reset by sm_gather)
    S.nred = 0u;
  }
  __syncthreads();
  if (t == 0) {
    S.vis[src >> 5] |= 1u << (src & 31u);
    S.front[src >> 5] |= 1u << (src & 31u);
  }
  cl.sync();  // every -1 store is ordered before the source's entry
  if (c == 0 && t == 0) {
    P.ctrl->ts[0] = globaltimer();
#if GK_SM_TRACE
    P.ctrl->ts[0] = t_entry;
#endif
    P.ctrl->tag[0] = kTagInit;
    P.parent[src] = (int32_t)src;
    if (P.want_depth) P.depth[src] = 0;
  }

  SM_MARK('i');
  long long etc = P.m;                                    // bfs.hpp:139
  long long scout = offv(P, P.out_off, src + 1) - offv(P, P.out_off, src);  // bfs.hpp:140
  long long fsz = 1, nsteps = 0;
  int lvl = 0;
  unsigned L = 0;  // levels done (parity of the slice / counter buffers)

  // the frontier list of the coming top-down level was gathered with the
  // last level's slices (ids, offsets, degree prefix in ids / off / pre)
  bool have_list = false;
  // every CTA passed the last level's cluster barrier and gather (false after
  // redundant levels: the slices are re-zeroed between two barriers first)
  bool synced = true;
  while (fsz > 0) {  // bfs.hpp:142
    if (P.strategy == GK_BFS_DIRECTION_OPTIMIZING && scout > etc / P.alpha) {
      long long awake = fsz, old_awake;  // bfs.hpp:146
      do {                               // bfs.hpp:149-154
        old_awake = awake;
        sm_resync(S, cl, synced, wlo, whi);
        const int q3 = (int)(L % 3u);
        // ---- bottom-up over this CTA's pending vertices (slice[q3] is zero) ----
        if (t == 0) S.nlong = 0u;
        const int k = sm_list<true>(S, S.vis, wlo, whi, rs);  // (sm_list ends with a CTA barrier)
        SM_MARK('p');
        // the pending vertices' in-offsets into shared memory (one round
        // trip for all of them), then kSmBuW slots per thread over this
        // thread's entries (i = t mod kSmBlock): a slot whose vertex resolves
        // (or is deferred) takes the next entry at once
        for (int i = t; i < k; i += kSmBlock) {
          const uint32_t v = S.ids[i];
          S.off[i] = (uint32_t)offv(P, P.in_off, v);
          S.pre[i] = (uint32_t)offv(P, P.in_off, v + 1);
        }
        __syncthreads();
        uint32_t* longl = reinterpret_cast<uint32_t*>(&S.wl[0][0]);  // free during bottom-up levels
        {
          uint32_t v[kSmBuW], b[kSmBuW], e[kSmBuW], rounds[kSmBuW];
          bool live[kSmBuW];
          int nexti = t;
#pragma unroll
          for (int q = 0; q < kSmBuW; q++) {
            live[q] = nexti < k;
            v[q] = b[q] = e[q] = rounds[q] = 0u;
            if (live[q]) {
              v[q] = S.ids[nexti];
              b[q] = S.off[nexti];
              e[q] = S.pre[nexti];
              nexti += kSmBlock;
            }
          }
          for (;;) {
            bool any = false;
#pragma unroll
            for (int q = 0; q < kSmBuW; q++) any |= live[q];
            if (!any) break;
            uint32_t u[kSmBuW][kSmBuR];
#pragma unroll
            for (int q = 0; q < kSmBuW; q++)
#pragma unroll
              for (int j = 0; j < kSmBuR; j++)
                u[q][j] = (live[q] && b[q] + j < e[q]) ? ld_nb(P.in_nb + b[q] + j) : kNoVertex;
#pragma unroll
            for (int q = 0; q < kSmBuW; q++) {
              if (!live[q]) continue;
              int hit = -1;
#pragma unroll
              for (int j = kSmBuR - 1; j >= 0; j--)
                if (u[q][j] != kNoVertex && sm_bit(S.front, u[q][j])) hit = j;
              bool done = false;
              if (hit >= 0) {  // the first in-neighbour in the frontier (bfs.hpp:55-60)
                uint32_t par = u[q][0];
#pragma unroll
                for (int j = 1; j < kSmBuR; j++)
                  if (hit == j) par = u[q][j];
                P.parent[v[q]] = (int32_t)par;
                if (P.want_depth) P.depth[v[q]] = lvl + 1;
                atomicOr(&S.slice[q3][(v[q] >> 5) - wlo], 1u << (v[q] & 31u));
                done = true;
              } else {
                b[q] += kSmBuR;
                if (b[q] >= e[q]) {
                  done = true;  // whole list scanned: not reached at this level
                } else if (++rounds[q] == kSmRounds) {
                  longl[atomicAdd(&S.nlong, 1u)] = v[q];  // resumes at in_off + kSmBuR * kSmRounds
                  done = true;
                }
              }
              if (done) {  // next entry of this thread
                live[q] = nexti < k;
                if (live[q]) {
                  v[q] = S.ids[nexti];
                  b[q] = S.off[nexti];
                  e[q] = S.pre[nexti];
                  rounds[q] = 0u;
                  nexti += kSmBlock;
                }
              }
            }
          }
        }
        __syncthreads();
        SM_MARK('q');
        const int nl = (int)S.nlong;
        for (int i = (int)warp; i < nl; i += kSmWarps) {  // long lists: a warp per vertex
          const uint32_t v = longl[i];
          const int64_t le = offv(P, P.in_off, v + 1);
          for (int64_t j = offv(P, P.in_off, v) + kSmBuR * kSmRounds; j < le; j += 32) {
            const int64_t jj = j + lane;
            uint32_t u = 0;
            bool h = false;
            if (jj < le) {
              u = ld_nb(P.in_nb + jj);
              h = sm_bit(S.front, u);
            }
            const unsigned bal = __ballot_sync(kFull, h);
            if (bal) {
              const uint32_t hu = __shfl_sync(kFull, u, __ffs(bal) - 1);
              if (lane == 0) {
                P.parent[v] = (int32_t)hu;
                if (P.want_depth) P.depth[v] = lvl + 1;
                atomicOr(&S.slice[q3][(v >> 5) - wlo], 1u << (v & 31u));
              }
              break;
            }
          }
        }
        __syncthreads();
        unsigned mine = 0;
        for (int j = t; j < whi - wlo; j += kSmBlock) {
          mine += __popc(S.slice[q3][j]);
          S.slice[(q3 + 1) % 3][j] = 0u;  // the next level's slice (last read two levels ago)
        }
        mine = sm_sum3(mine, 0u, 0u, S, rs).x;
        sm_push(S, cl, C, c, q3, make_uint4(mine, 0u, 1u, 0u));  // no won lists after a bottom-up step
        SM_MARK('r');
        cl.sync();
        SM_MARK('s');
        awake = sm_totals(S, C, q3).cnt;
        sm_gather(S, cl, C, W, Wc, q3, false, 0, 0, rs);
        SM_MARK('t');
        L++;
        sm_log(P, c, nsteps++, 'B', old_awake, awake, etc);
        lvl++;
      } while (awake >= old_awake || awake > P.n / P.beta);
      fsz = awake;
      scout = 1;  // bfs.hpp:156
      have_list = false;
    } else {
      etc -= scout;  // bfs.hpp:158
      const int q3 = (int)(L % 3u), wp = (int)(L & 1u);
      // Small frontiers (<= kSmWon vertices): every CTA lists the whole
      // frontier and takes 1/C of its edges; claims go straight to the
      // target's owner over DSMEM (one cluster barrier per level).  Larger
      // ones: each CTA expands its own slice, claims in a local bitmap, and
      // the owners merge the C copies (two barriers, no per-claim traffic).
      const bool fewer = fsz <= kSmWon;  // uniform: fsz is a cluster total
      int k;
      if (have_list) {  // the C won lists of the last level, gathered after its barrier
        k = (int)fsz;
      } else {  // from the replicated front: all of it, or this CTA's slice
        k = fewer ? sm_list<false>(S, S.front, 0, W, rs) : sm_list<false>(S, S.front, wlo, whi, rs);
        for (int i = t; i < k; i += kSmBlock) {
          const uint32_t v = S.ids[i];
          const int64_t o0 = offv(P, P.out_off, v), o1 = offv(P, P.out_off, v + 1);
          S.off[i] = (uint32_t)o0;
          S.pre[i] = (uint32_t)(o1 - o0);
        }
      }
      SM_MARK('a');
      const long long E = have_list ? (long long)S.pre[k]  // the gather's (or last level's) scan wrote the prefix
                                    : sm_prefix(S, k, rs);
      SM_MARK('b');
      if (k == fsz && E <= kSmRedE) {  // uniform: the whole frontier is listed in every CTA
        // ---- redundant level: every CTA expands the whole frontier against
        // its own copy of visited (the copies are identical), so every CTA
        // claims the same set; the owner of a claimed vertex stores its
        // parent (one writer).  No cluster barrier, no DSMEM ----
        for (long long eb = t; eb < E; eb += kSmTdW * kSmBlock) {
          uint32_t u[kSmTdW], w[kSmTdW];
          bool ok[kSmTdW];
#pragma unroll
          for (int q = 0; q < kSmTdW; q++) {
            const long long e = eb + (long long)q * kSmBlock;
            ok[q] = e < E;
            u[q] = w[q] = 0u;
            if (ok[q]) {
              int lo = 0, hi = k;
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if ((long long)S.pre[mid] <= e) lo = mid;
                else hi = mid;
              }
              u[q] = S.ids[lo];
              w[q] = ld_nb(P.out_nb + (S.off[lo] + (uint32_t)(e - S.pre[lo])));
            }
          }
#pragma unroll
          for (int q = 0; q < kSmTdW; q++) {
            if (!ok[q] || sm_bit(S.vis, w[q]) || sm_bit(S.nxt, w[q])) continue;
            const uint32_t bit = 1u << (w[q] & 31u), ww = w[q] >> 5;
            if (!(atomicOr(&S.nxt[ww], bit) & bit)) {
              if ((int)ww >= wlo && (int)ww < whi) P.parent[w[q]] = (int32_t)u[q];  // bfs.hpp:77-84
              S.front[atomicAdd(&S.nred, 1u)] = w[q];  // the new frontier, listed (<= E <= kSmMaxW)
            }
          }
        }
        __syncthreads();
        SM_MARK('1');
        // the new frontier (every vertex claimed here was unvisited): its
        // list with offsets and degrees for the next level, the counters
        const int kn = (int)S.nred;
        SM_MARK('2');
        unsigned scl = 0;
        for (int i = t; i < kn; i += kSmBlock) {
          const uint32_t v = S.front[i];
          S.ids[i] = v;
          const int64_t o0 = offv(P, P.out_off, v), o1 = offv(P, P.out_off, v + 1);
          const uint32_t dg = (uint32_t)(o1 - o0);
          S.off[i] = (uint32_t)o0;
          S.pre[i] = dg;
          scl += encode ? (dg ? dg : 1u) : dg;  // -old of bfs.hpp:83 / the rescan pass of bfs.hpp:161-167
          const int vw = (int)(v >> 5);
          if (P.want_depth && vw >= wlo && vw < whi) P.depth[v] = lvl + 1;
        }
        scl = sm_sum3(scl, 0u, 0u, S, rs).x;  // (every read of the list in front is done)
        if (t == 0) S.nred = 0u;
        SM_MARK('3');
        for (int j = 4 * t; j < W; j += 4 * kSmBlock) {
          const uint4 x = *reinterpret_cast<const uint4*>(&S.nxt[j]);
          uint4 v = *reinterpret_cast<const uint4*>(&S.vis[j]);
          v.x |= x.x;
          v.y |= x.y;
          v.z |= x.z;
          v.w |= x.w;
          *reinterpret_cast<uint4*>(&S.vis[j]) = v;
          *reinterpret_cast<uint4*>(&S.front[j]) = x;
          *reinterpret_cast<uint4*>(&S.nxt[j]) = make_uint4(0u, 0u, 0u, 0u);
        }
        SM_MARK('4');
        const long long e_next = sm_prefix(S, kn, rs);
        SM_MARK('5');
        L++;
        const long long fsize = fsz;
        fsz = kn;
        scout = scl;
        // the list is in this CTA's claim order: good for a redundant level
        // (every CTA expands all of it); a cluster-wide level splits the
        // edges by position, which needs the same order everywhere -- it
        // lists the front bitmap instead
        have_list = e_next <= kSmRedE;
        synced = false;
        sm_log(P, c, nsteps++, 'T', fsize, scout, etc);
        lvl++;
        continue;
      }
      sm_resync(S, cl, synced, wlo, whi);
      // ---- claims (bfs.hpp:77-84) ----
      const long long e0 = fewer ? E * c / C : 0, e1 = fewer ? E * (c + 1) / C : E;
      long long cc = 0, sc = 0;
      bool ovf = false;
      for (long long eb = e0 + t; eb < e1; eb += kSmTdW * kSmBlock) {
        uint32_t u[kSmTdW], w[kSmTdW];
        bool ok[kSmTdW];
#pragma unroll
        for (int q = 0; q < kSmTdW; q++) {
          const long long e = eb + (long long)q * kSmBlock;
          ok[q] = e < e1;
          u[q] = 0u;
          w[q] = 0u;
          if (ok[q]) {
            int lo = 0, hi = k;  // last entry with pre[i] <= e (its range holds e)
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if ((long long)S.pre[mid] <= e) lo = mid;
              else hi = mid;
            }
            u[q] = S.ids[lo];
            w[q] = ld_nb(P.out_nb + (S.off[lo] + (uint32_t)(e - S.pre[lo])));
          }
        }
        // first attempt on this target from this CTA (local claim bitmap)
#pragma unroll
        for (int q = 0; q < kSmTdW; q++) {
          if (ok[q] && !sm_bit(S.vis, w[q]) && !sm_bit(S.nxt, w[q])) {
            const uint32_t bit = 1u << (w[q] & 31u);
            ok[q] = !(atomicOr(&S.nxt[w[q] >> 5], bit) & bit);
          } else {
            ok[q] = false;
          }
        }
        if (!fewer) {  // large frontier: the local claimer stores a (valid) parent; owners merge later
#pragma unroll
          for (int q = 0; q < kSmTdW; q++)
            if (ok[q]) P.parent[w[q]] = (int32_t)u[q];
          continue;
        }
        // small frontier: the owner's slice decides the one winner, which
        // stores the parent, keeps the degree (read with the claim) and
        // lists the vertex for the next level
        int64_t o0[kSmTdW], o1[kSmTdW];
        uint32_t old[kSmTdW];
#pragma unroll
        for (int q = 0; q < kSmTdW; q++) {
          o0[q] = o1[q] = 0;
          old[q] = ~0u;
          if (ok[q]) {
            const uint32_t ww = w[q] >> 5;
            const int home = (int)(ww / (uint32_t)Wc);
            o0[q] = offv(P, P.out_off, w[q]);
            o1[q] = offv(P, P.out_off, w[q] + 1);
            old[q] = atomicOr(cl.map_shared_rank(&S.slice[q3][0], home) + (ww - (uint32_t)home * (uint32_t)Wc),
                              1u << (w[q] & 31u));
          }
        }
#pragma unroll
        for (int q = 0; q < kSmTdW; q++) {
          if (!ok[q] || ((old[q] >> (w[q] & 31u)) & 1u)) continue;
          P.parent[w[q]] = (int32_t)u[q];
          if (P.want_depth) P.depth[w[q]] = lvl + 1;
          const long long dg = o1[q] - o0[q];
          sc += encode ? (dg ? dg : 1) : dg;  // -old of bfs.hpp:83 / the rescan pass of bfs.hpp:161-167
          cc++;
          const unsigned i = atomicAdd(&S.nwon, 1u);
          if (i < (unsigned)kSmWon) {
            S.wl[wp][i] = make_uint4(w[q], (uint32_t)o0[q], (uint32_t)dg, 0u);
          } else {
            ovf = true;
          }
        }
      }
      SM_MARK('c');
      if (!fewer) {
        cl.sync();  // every CTA's attempts are in its claim bitmap
        SM_MARK('d');
        // merge this CTA's slice of the C claim bitmaps (all C loads in flight)
        for (int j = wlo + 4 * t; j < whi; j += 4 * kSmBlock) {  // 16-byte DSMEM loads, C in flight
          uint4 x = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 1
          for (int r0 = 0; r0 < C; r0 += 8) {
            uint4 y[8];
#pragma unroll
            for (int r = 0; r < 8; r++)
              y[r] = r0 + r < C ? *reinterpret_cast<const uint4*>(cl.map_shared_rank(&S.nxt[0], r0 + r) + j)
                                : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int r = 0; r < 8; r++) {
              x.x |= y[r].x;
              x.y |= y[r].y;
              x.z |= y[r].z;
              x.w |= y[r].w;
            }
          }
          const uint4 v = *reinterpret_cast<const uint4*>(&S.vis[j]);
          *reinterpret_cast<uint4*>(&S.slice[q3][j - wlo]) =
              make_uint4(x.x & ~v.x, x.y & ~v.y, x.z & ~v.z, x.w & ~v.w);
        }
        __syncthreads();
        SM_MARK('e');
        const int kn = sm_list<false>(S, S.slice[q3], 0, whi - wlo, rs);  // ids relative to wlo * 32
        for (int i = t; i < kn; i += kSmBlock) {
          const uint32_t v = S.ids[i] + (uint32_t)wlo * 32u;
          const int64_t o0 = offv(P, P.out_off, v), o1 = offv(P, P.out_off, v + 1);
          const long long dg = o1 - o0;
          sc += encode ? (dg ? dg : 1) : dg;
          if (P.want_depth) P.depth[v] = lvl + 1;
          if (i < kSmWon) {  // this CTA's share of the next frontier
            S.wl[wp][i] = make_uint4(v, (uint32_t)o0, (uint32_t)dg, 0u);
          }
        }
        cc = kn;
        ovf = kn > kSmWon;
        if (t == 0) S.nwon = (unsigned)kn;
      }
      for (int j = t; j < whi - wlo; j += kSmBlock) S.slice[(q3 + 1) % 3][j] = 0u;
      const uint3 sums = sm_sum3(fewer ? (unsigned)cc : 0u, (unsigned)sc, ovf ? 1u : 0u, S, rs);
      if (fewer) cc = sums.x;
      sc = sums.y;
      const unsigned ovf_any = sums.z;
      __syncthreads();  // S.nwon final
      sm_push(S, cl, C, c, q3, make_uint4((unsigned)cc, (unsigned)sc, ovf_any ? 1u : 0u, min(S.nwon, (unsigned)kSmWon)));
      SM_MARK('f');
      cl.sync();  // every claim has landed in its owner's slice
      SM_MARK('g');
      const SmTot tt = sm_totals(S, C, q3);
      // the next level's direction (the test at the top of the loop, same
      // totals): a top-down level over a small frontier takes the won lists
      // now, in the slices' round trip
      const bool next_td = !(P.strategy == GK_BFS_DIRECTION_OPTIMIZING && tt.sc > etc / P.alpha);
      have_list = next_td && tt.lists && tt.cnt > 0 && tt.cnt <= kSmWon;
      sm_gather(S, cl, C, W, Wc, q3, have_list, wp, (int)tt.cnt, rs);
      SM_MARK('h');
      L++;
      const long long fsize = fsz;
      fsz = tt.cnt;
      scout = tt.sc;
      sm_log(P, c, nsteps++, 'T', fsize, scout, etc);
      lvl++;
    }
  }
  if (c == 0 && t == 0) P.ctrl->num_steps = nsteps;
#if GK_SM_SPAN
  if (c == 0 && t == 0) {
    P.ctrl->ts[510] = t_in;
    P.ctrl->ts[511] = globaltimer();
    P.ctrl->tag[510] = P.ctrl->tag[511] = 'x';
  }
#endif
  // bfs.hpp:171-175's final sweep: unreached slots were written -1 at init.
  // No CTA may exit while a peer can still read its shared memory.
  cl.sync();
}

}  // namespace

// Cluster size for graphs with n <= 8192 x cluster (0: the small-graph
// kernel is not used for this graph / device).  m < 2^32 keeps offsets in
// 32 bits; the bound 2^25 keeps the regime where one cluster beats the grid.
cudaError_t small_configure(int device, int64_t n, int64_t m, int* cluster) {
  *cluster = 0;
  if (n < 1 || m > (int64_t(1) << 25) || n > (int64_t)kSmMaxW * 32) return cudaSuccess;
  cudaError_t e;
  const size_t smem = sizeof(SmShared);
  if ((e = cudaFuncSetAttribute(bfs_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  cudaFuncSetAttribute(bfs_small, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  const int64_t w = (n + 31) / 32;
  int cs_max = 16;
  if (const char* e = getenv("GK_SM_CLUSTER")) cs_max = atoi(e) >= 16 ? 16 : 8;  // A/B
  for (int cs = cs_max; cs >= 8; cs /= 2) {
    if ((((w + cs - 1) / cs + 3) & ~int64_t(3)) > kSmSlice) break;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kSmBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (void*)bfs_small, &cfg) == cudaSuccess && nc >= 1) {
      *cluster = cs;
      return cudaSuccess;
    }
    cudaGetLastError();
  }
  (void)device;
  return cudaSuccess;
}

cudaError_t small_launch(const BfsParams& p, int cluster, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kSmBlock);
  cfg.dynamicSmemBytes = sizeof(SmShared);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, bfs_small, p);
}

}  // namespace gk
