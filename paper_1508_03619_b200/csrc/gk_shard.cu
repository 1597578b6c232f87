// gk_shard.cu -- one rank's part of the 1D-partitioned BFS.
//
// Vertex v is owned by rank v / block (block = ceil(n/P) rounded up to a
// multiple of 32 so every rank's slice of a bitmap is whole words).  A rank
// stores the CSR rows of its owned vertices (global neighbour ids), their
// parent / visited state, and its local frontier queue.  The host
// orchestrator (paper_1508_03619_b200/dist.py) runs the reference's level
// loop (bfs.hpp:139-169) and performs the exchanges between these kernels:
//   top-down  : expand the owned frontier; owned targets are claimed in place,
//               remote targets become (v, u) pairs bucketed by owner (deduped
//               per level with a sent-bitmap) -> all-to-all -> td_apply
//   bottom-up : owned unvisited vertices scan their in-lists against the
//               replicated n-bit front bitmap; the owned slice of `next` is
//               then all-gathered
// The single-GPU path is the persistent kernel in gk_bfs_kernel.cu; this file
// is the multi-GPU path, launched per phase on a caller-provided stream so
// the exchanges (NCCL through torch.distributed) order with the kernels.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr int kSB = 512;             // block size of the shard kernels
constexpr int64_t kShHeavy = 1024;   // degree above which a vertex is chunked
constexpr int kShChunk = 1024;
constexpr unsigned kFullMask = 0xffffffffu;

// device counter slots
enum : int { cTail = 0, cPairs = 1, cScout = 2, cClaims = 3, cAwake = 4, cChunks = 5, cLong = 6, cDest = 8 };

struct ShardParams {
  int64_t n, lo, hi, nloc, block;
  int rank, nranks;
  const int64_t* off;
  const uint32_t* nb;
  int32_t* parent;
  int32_t* depth;
  uint32_t* visited;  // local, nloc bits
  uint32_t* sent;     // global n bits: remote targets already sent this level
  uint32_t* queue;
  uint64_t* pairs;    // outbox (unsorted)
  uint64_t* pairs_out;
  int64_t pair_cap;
  Chunk* chunks;
  int64_t chunk_cap;
  unsigned long long* ctr;
  int want_depth;
  int encode;
  int dedup;  // use (and set) the sent bitmap this level
  int big;    // large top-down step: owned claims go to `next`, then k_sh_sweep
  uint32_t* next;        // owned next bitmap (big top-down steps), starts as visited
  const uint32_t* dead;  // owned never-reachable bitmap
  uint32_t* longq;       // bottom-up long-list scratch (aliases pairs)
  int64_t long_cap;
};

__device__ __forceinline__ unsigned lmask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Warp-aggregated append of one value per active lane into arr at *cursor.
template <typename T>
__device__ __forceinline__ void warp_append(bool want, T val, T* arr, unsigned long long* cursor,
                                            int64_t cap, int* overflow) {
  const unsigned m = __ballot_sync(kFullMask, want);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cursor, (unsigned long long)__popc(m));
  base = __shfl_sync(kFullMask, base, leader);
  if (want) {
    const unsigned long long pos = base + __popc(m & lmask_lt());
    if ((int64_t)pos < cap) arr[pos] = val;
    else *overflow = 1;
  }
}

__device__ __forceinline__ long long local_degree(const ShardParams& P, uint32_t v) {
  const int64_t r = (int64_t)v - P.lo;
  return P.off[r + 1] - P.off[r];
}

// ---- per-warp append buffers (QueueBuffer analogue, sliding_queue.hpp:62-86)
constexpr int kQB = 256;  // queue entries per warp buffer
constexpr int kPB = 128;  // remote pairs per warp buffer

__device__ __forceinline__ void flush_q(const ShardParams& P, uint32_t* buf, int& n, int* overflow) {
  __syncwarp();
  if (n == 0) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&P.ctr[cTail], (unsigned long long)n);
  base = __shfl_sync(kFullMask, base, 0);
  for (int i = lane; i < n; i += 32) {
    if ((int64_t)(base + i) < P.nloc + 1) P.queue[base + i] = buf[i];
    else *overflow = 1;
  }
  __syncwarp();
  n = 0;
}
__device__ __forceinline__ void push_q(const ShardParams& P, bool want, uint32_t v, uint32_t* buf, int& n,
                                       int* overflow) {
  const unsigned m = __ballot_sync(kFullMask, want);
  if (!m) return;
  if (want) buf[n + __popc(m & lmask_lt())] = v;
  n += __popc(m);
  if (n > kQB - 32) flush_q(P, buf, n, overflow);
}
__device__ __forceinline__ void flush_p(const ShardParams& P, uint64_t* buf, int& n, int* overflow) {
  __syncwarp();
  if (n == 0) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&P.ctr[cPairs], (unsigned long long)n);
  base = __shfl_sync(kFullMask, base, 0);
  for (int i = lane; i < n; i += 32) {
    if ((int64_t)(base + i) < P.pair_cap) P.pairs[base + i] = buf[i];
    else *overflow = 1;
  }
  __syncwarp();
  n = 0;
}
__device__ __forceinline__ void push_p(const ShardParams& P, bool want, uint64_t pr, uint64_t* buf, int& n,
                                       int* overflow) {
  const unsigned m = __ballot_sync(kFullMask, want);
  if (!m) return;
  if (want) buf[n + __popc(m & lmask_lt())] = pr;
  n += __popc(m);
  if (n > kPB - 32) flush_p(P, buf, n, overflow);
}

struct WarpBufs {
  uint32_t* q;
  uint64_t* p;
  int qn, pn;
};

// N edges (u_k -> v_k) per thread, loads and atomics of all N issued
// together.  Owned targets: small steps claim with a visited pre-check +
// atomicOr (bfs.hpp:78-84) and append to the owned queue; big steps
// (P.big) only store a parent and RED the bit into the owned next-bitmap
// (which starts as a copy of visited), leaving degrees and the queue to
// the claim sweep.  Remote targets become (v, u) pairs for their owner,
// deduplicated per level through the sent-bitmap when P.dedup.
template <int N>
__device__ __forceinline__ void td_edges(const ShardParams& P, const uint32_t (&u)[N], const uint32_t (&v)[N],
                                         int lvl, long long& scout, long long& claims, WarpBufs& wb,
                                         int* overflow) {
  bool loc[N], rem[N];
  uint32_t w[N];
#pragma unroll
  for (int k = 0; k < N; k++) {
    const bool ok = v[k] != kNoVertex;
    loc[k] = ok && (int64_t)v[k] >= P.lo && (int64_t)v[k] < P.hi;
    rem[k] = ok && !loc[k];
    w[k] = 0xffffffffu;
    if (loc[k]) {
      const uint32_t r = (uint32_t)((int64_t)v[k] - P.lo);
      w[k] = __ldcg((P.big ? P.next : P.visited) + (r >> 5));
    } else if (rem[k] && P.dedup) {
      w[k] = __ldcg(P.sent + (v[k] >> 5));
    }
  }
#pragma unroll
  for (int k = 0; k < N; k++) {
    if (loc[k]) {
      const uint32_t r = (uint32_t)((int64_t)v[k] - P.lo);
      const uint32_t bit = 1u << (r & 31u);
      if (P.big) {
        if (!(w[k] & bit)) {
          P.parent[r] = (int32_t)u[k];
          atomicOr(P.next + (r >> 5), bit);  // result unused -> RED
        }
        loc[k] = false;
      } else {
        loc[k] = !(w[k] & bit) && !(atomicOr(P.visited + (r >> 5), bit) & bit);
      }
    } else if (rem[k] && P.dedup) {
      const uint32_t bit = 1u << (v[k] & 31u);
      rem[k] = !(w[k] & bit) && !(atomicOr(P.sent + (v[k] >> 5), bit) & bit);
    }
  }
#pragma unroll
  for (int k = 0; k < N; k++) {
    if (loc[k]) {
      const uint32_t r = (uint32_t)((int64_t)v[k] - P.lo);
      P.parent[r] = (int32_t)u[k];
      if (P.want_depth) P.depth[r] = lvl + 1;
      if (P.encode) {
        const long long d = local_degree(P, v[k]);
        scout += d ? d : 1;  // -old of the degree-encoded slot (bfs.hpp:83)
      } else {
        scout += 1;
      }
      claims++;
    }
  }
#pragma unroll
  for (int k = 0; k < N; k++) {
    push_q(P, loc[k], v[k], wb.q, wb.qn, overflow);
    push_p(P, rem[k], ((uint64_t)v[k] << 32) | u[k], wb.p, wb.pn, overflow);
  }
}

__device__ void block_sum2(long long a, long long b, unsigned long long* da, unsigned long long* db) {
  __shared__ long long red[2][kSB / 32];
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(kFullMask, a, o);
    b += __shfl_down_sync(kFullMask, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long ta = 0, tb = 0;
    for (int i = 0; i < kSB / 32; i++) {
      ta += red[0][i];
      tb += red[1][i];
    }
    if (ta) atomicAdd(da, (unsigned long long)ta);
    if (tb) atomicAdd(db, (unsigned long long)tb);
  }
}

// parent := -1, visited := the owned dead bitmap (never-reachable vertices)
__global__ void k_sh_init(ShardParams P) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < P.nloc; i += gs) {
    P.parent[i] = -1;
    if (P.want_depth) P.depth[i] = -1;
  }
  for (long long i = gt; i < (P.nloc + 31) / 32; i += gs) P.visited[i] = __ldg(P.dead + i);
}

__global__ void k_sh_set_source(ShardParams P, uint32_t src) {
  const uint32_t r = (uint32_t)((int64_t)src - P.lo);
  P.parent[r] = (int32_t)src;
  if (P.want_depth) P.depth[r] = 0;
  P.visited[r >> 5] |= 1u << (r & 31u);
  P.queue[0] = src;
  P.ctr[cTail] = 1;
}

__global__ void k_sh_copy_words(const uint32_t* src, uint32_t* dst, long long words) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}

// Top-down expansion of queue[qs, qe): tiles of kSB frontier vertices, CTA
// scan of degrees, load-balanced edge gather, 4 edges per thread in flight;
// vertices of degree > kShHeavy become kShChunk-edge chunks for
// k_sh_td_heavy.
__global__ void __launch_bounds__(kSB) k_sh_td_light(ShardParams P, unsigned long long qs, unsigned long long qe,
                                                     int lvl) {
  __shared__ int64_t t_b[kSB];
  __shared__ int64_t t_pre[kSB + 1];
  __shared__ uint32_t t_u[kSB];
  __shared__ int64_t wsum[kSB / 32 + 1];
  __shared__ uint32_t qbuf[kSB / 32][kQB];
  __shared__ uint64_t pbuf[kSB / 32][kPB];
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpBufs wb{qbuf[warp], pbuf[warp], 0, 0};
  long long scout = 0, claims = 0;
  for (unsigned long long tile = blockIdx.x; qs + tile * kSB < qe; tile += gridDim.x) {
    const unsigned long long i = qs + tile * kSB + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, dl = 0;
    if (i < qe) {
      u = __ldcg(P.queue + i);
      const int64_t r = (int64_t)u - P.lo;
      b = P.off[r];
      const int64_t d = P.off[r + 1] - b;
      if (d > kShHeavy) {
        const int64_t nch = (d + kShChunk - 1) / kShChunk;
        const unsigned long long base = atomicAdd(&P.ctr[cChunks], (unsigned long long)nch);
        if ((int64_t)(base + nch) <= P.chunk_cap) {
          for (int64_t c = 0; c < nch; c++) {
            Chunk ch;
            ch.u = u;
            ch.start = b + c * kShChunk;
            ch.len = (uint32_t)((d - c * kShChunk) < kShChunk ? (d - c * kShChunk) : kShChunk);
            P.chunks[base + c] = ch;
          }
        } else {
          overflow = 1;
        }
      } else {
        dl = d;
      }
    }
    int64_t incl = dl;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t run = 0;
      for (int w = 0; w < kSB / 32; w++) {
        const int64_t t = wsum[w];
        wsum[w] = run;
        run += t;
      }
      wsum[kSB / 32] = run;
    }
    __syncthreads();
    t_pre[threadIdx.x] = wsum[warp] + incl - dl;
    t_u[threadIdx.x] = u;
    t_b[threadIdx.x] = b;
    const int64_t tot = wsum[kSB / 32];
    __syncthreads();
    for (int64_t eb = 0; eb < tot; eb += 4 * kSB) {
      uint32_t uu[4], v[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int64_t ei = eb + k * kSB + threadIdx.x;
        uu[k] = 0;
        v[k] = kNoVertex;
        if (ei < tot) {
          int lo = 0, hi = kSB - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (t_pre[mid] <= ei) lo = mid;
            else hi = mid - 1;
          }
          uu[k] = t_u[lo];
          v[k] = __ldg(P.nb + t_b[lo] + (ei - t_pre[lo]));
        }
      }
      td_edges<4>(P, uu, v, lvl, scout, claims, wb, &overflow);
    }
    __syncthreads();
  }
  flush_q(P, wb.q, wb.qn, &overflow);
  flush_p(P, wb.p, wb.pn, &overflow);
  block_sum2(scout, claims, &P.ctr[cScout], &P.ctr[cClaims]);
  if (threadIdx.x == 0 && overflow) atomicExch((unsigned*)&P.ctr[7], 1u);
}

// Heavy chunks: static round-robin over warps, 8 edges per lane in flight.
__global__ void __launch_bounds__(kSB) k_sh_td_heavy(ShardParams P, unsigned long long nch, int lvl) {
  __shared__ uint32_t qbuf[kSB / 32][kQB];
  __shared__ uint64_t pbuf[kSB / 32][kPB];
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpBufs wb{qbuf[warp], pbuf[warp], 0, 0};
  long long scout = 0, claims = 0;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (unsigned long long c = gw; c < nch; c += nw) {
    const Chunk ch = P.chunks[c];
    uint32_t uu[8];
#pragma unroll
    for (int k = 0; k < 8; k++) uu[k] = ch.u;
    for (uint32_t o = 0; o < ch.len; o += 256) {
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint32_t j = o + lane + 32u * k;
        v[k] = j < ch.len ? __ldg(P.nb + ch.start + j) : kNoVertex;
      }
      td_edges<8>(P, uu, v, lvl, scout, claims, wb, &overflow);
    }
  }
  flush_q(P, wb.q, wb.qn, &overflow);
  flush_p(P, wb.p, wb.pn, &overflow);
  block_sum2(scout, claims, &P.ctr[cScout], &P.ctr[cClaims]);
  if (threadIdx.x == 0 && overflow) atomicExch((unsigned*)&P.ctr[7], 1u);
}

// Bucket the outbox by owner rank: count, then scatter into pairs_out at
// per-destination offsets (exclusive scan done on the host, P is small).
// Both passes aggregate per CTA in shared memory (one global atomic per
// CTA and destination: per-pair atomics on P counters serialise).
constexpr int kMaxRanksSmem = 64;
__global__ void __launch_bounds__(kSB) k_sh_count_dest(ShardParams P, unsigned long long npairs) {
  __shared__ unsigned hist[kMaxRanksSmem];
  for (int i = threadIdx.x; i < P.nranks; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < npairs;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)(P.pairs[i] >> 32);
    atomicAdd(&hist[(int)((int64_t)v / P.block)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P.nranks; i += blockDim.x)
    if (hist[i]) atomicAdd(&P.ctr[cDest + i], (unsigned long long)hist[i]);
}
__global__ void __launch_bounds__(kSB) k_sh_scatter_dest(ShardParams P, unsigned long long npairs,
                                                         unsigned long long* cursor) {
  __shared__ unsigned hist[kMaxRanksSmem];
  __shared__ unsigned long long base[kMaxRanksSmem];
  // contiguous slice of the outbox per CTA
  const unsigned long long per = (npairs + gridDim.x - 1) / gridDim.x;
  const unsigned long long b0 = per * blockIdx.x, b1 = b0 + per < npairs ? b0 + per : npairs;
  for (int i = threadIdx.x; i < P.nranks; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (unsigned long long i = b0 + threadIdx.x; i < b1; i += blockDim.x)
    atomicAdd(&hist[(int)((int64_t)(P.pairs[i] >> 32) / P.block)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < P.nranks; i += blockDim.x) {
    base[i] = hist[i] ? atomicAdd(&cursor[i], (unsigned long long)hist[i]) : 0ull;
    hist[i] = 0;
  }
  __syncthreads();
  for (unsigned long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const uint64_t pr = P.pairs[i];
    const int d = (int)((int64_t)(pr >> 32) / P.block);
    P.pairs_out[base[d] + atomicAdd(&hist[d], 1u)] = pr;
  }
}

// Received (v, u) pairs: claim owned v (same two modes as td_edges).
__global__ void __launch_bounds__(kSB) k_sh_td_apply(ShardParams P, const uint64_t* in, unsigned long long npairs,
                                                     int lvl) {
  __shared__ uint32_t qbuf[kSB / 32][kQB];
  __shared__ uint64_t pbuf[kSB / 32][kPB];
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  WarpBufs wb{qbuf[warp], pbuf[warp], 0, 0};
  long long scout = 0, claims = 0;
  const unsigned long long stride = 4ull * gridDim.x * blockDim.x;
  const unsigned long long base = 4ull * blockIdx.x * blockDim.x;
  for (unsigned long long i0 = 0; i0 < npairs; i0 += stride) {
    uint32_t u[4], v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const unsigned long long i = i0 + base + (unsigned long long)k * blockDim.x + threadIdx.x;
      u[k] = 0;
      v[k] = kNoVertex;
      if (i < npairs) {
        const uint64_t pr = in[i];
        v[k] = (uint32_t)(pr >> 32);
        u[k] = (uint32_t)pr;
      }
    }
    td_edges<4>(P, u, v, lvl, scout, claims, wb, &overflow);
  }
  flush_q(P, wb.q, wb.qn, &overflow);
  block_sum2(scout, claims, &P.ctr[cScout], &P.ctr[cClaims]);
  if (threadIdx.x == 0 && overflow) atomicExch((unsigned*)&P.ctr[7], 1u);
}

// Claim sweep after a big top-down step (the owned analogue of the
// persistent kernel's td_scout_bits): a warp takes 32 owned words; claims =
// next & ~visited are folded into visited and appended to the queue in
// vertex order (one fetch-add per warp), and their degrees are read as
// sorted offset runs for scout.
__global__ void __launch_bounds__(kSB) k_sh_sweep(ShardParams P, int lvl) {
  __shared__ int overflow;
  if (threadIdx.x == 0) overflow = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long w32 = (P.nloc + 31) / 32;
  long long scout = 0, claims = 0;
  for (long long w0 = gw * 32; w0 < w32; w0 += nw * 32) {
    const long long w = w0 + lane;
    uint32_t cl = 0;
    if (w < w32) {
      const uint32_t nx = __ldcg(P.next + w), vis = __ldcg(P.visited + w);
      cl = nx & ~vis;
      if (cl) P.visited[w] = vis | cl;
    }
    const int cnt = __popc(cl);
    claims += cnt;
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(kFullMask, incl, 31);
    if (total == 0) continue;
    unsigned long long qb = 0;
    if (lane == 0) qb = atomicAdd(&P.ctr[cTail], (unsigned long long)total);
    qb = __shfl_sync(kFullMask, qb, 0);
    {
      uint32_t m = cl;
      unsigned long long q = qb + excl;
      while (m) {
        const int bp = __ffs(m) - 1;
        m &= m - 1;
        if ((int64_t)q < P.nloc + 1) P.queue[q] = (uint32_t)(P.lo + w * 32 + bp);
        else overflow = 1;
        q++;
      }
    }
    for (int base = 0; base < total; base += 128) {
      int64_t o0[4], o1[4], r[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int c = base + k * 32 + lane;
        int lo = 0;  // word holding the c-th claim: last lane with excl <= c
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int e = __shfl_sync(kFullMask, excl, lo + step);
          if (e <= c) lo += step;
        }
        const uint32_t m = __shfl_sync(kFullMask, cl, lo);
        const int ex = __shfl_sync(kFullMask, excl, lo);
        r[k] = -1;
        o0[k] = o1[k] = 0;
        if (c < total) {
          r[k] = (w0 + lo) * 32 + (int)__fns(m, 0, c - ex + 1);
          o0[k] = __ldg(P.off + r[k]);
          o1[k] = __ldg(P.off + r[k] + 1);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (r[k] < 0) continue;
        const long long d = o1[k] - o0[k];
        scout += P.encode ? (d ? d : 1) : 1;
        if (P.want_depth) P.depth[r[k]] = lvl + 1;
      }
    }
  }
  block_sum2(scout, claims, &P.ctr[cScout], &P.ctr[cClaims]);
  if (threadIdx.x == 0 && overflow) atomicExch((unsigned*)&P.ctr[7], 1u);
}

// Owned slice of the front bitmap from queue[qs, qe) (QueueToBitmap).
__global__ void k_sh_q2b(ShardParams P, unsigned long long qs, unsigned long long qe, uint32_t* slice) {
  for (unsigned long long i = qs + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < qe;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)((int64_t)__ldcg(P.queue + i) - P.lo);
    atomicOr(slice + (r >> 5), 1u << (r & 31u));
  }
}

// Bottom-up sweep of the owned vertices against the replicated front
// (bfs.hpp:47-66), the persistent kernel's bu_step on owned rows: a warp
// task is 32 owned words; pending (not visited, not dead) vertices are
// numbered by a warp prefix sum; 2 slots per lane refilled as they resolve,
// each round tests 4 in-neighbours of the list; after kShRounds rounds a
// vertex is deferred to k_sh_bu_long.
// Parent = first in-neighbour (ascending) with its front bit, as the
// reference picks.
constexpr int kShSlots = 2;
constexpr int kShRounds = 8;
__global__ void __launch_bounds__(kSB) k_sh_bu(ShardParams P, const uint32_t* front, uint32_t* next_slice, int lvl) {
  __shared__ uint32_t acc_all[kSB / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* acc = acc_all[warp];
  long long awake = 0;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long w32 = (P.nloc + 31) / 32;
  int tw_log = 5;  // task = 2^tw_log words, smaller when that leaves warps idle
  while (tw_log > 0 && ((w32 + (1 << tw_log) - 1) >> tw_log) < nw) tw_log--;
  const int tw = 1 << tw_log;
  const long long ntasks = (w32 + tw - 1) >> tw_log;
  for (long long t = gw; t < ntasks; t += nw) {
    const long long tbase = t << tw_log;
    const long long w = tbase + lane;
    uint32_t vis = 0xffffffffu, pad = 0u;
    if (lane < tw && w < w32) {
      vis = __ldcg(P.visited + w);
      const int64_t rem = P.nloc - w * 32;
      if (rem < 32) pad = 0xffffffffu << rem;
    }
    const uint32_t pm = ~(vis | pad);
    const int cnt = __popc(pm);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(kFullMask, incl, 31);
    acc[lane] = 0u;
    __syncwarp();
    int next_c = 0;
    uint32_t r[kShSlots], d[kShSlots], rounds[kShSlots];
    int64_t b[kShSlots];
    int st[kShSlots];  // 0 empty, 2 list rounds
#pragma unroll
    for (int k = 0; k < kShSlots; k++) {
      st[k] = 0;
      r[k] = d[k] = rounds[k] = 0;
      b[k] = 0;
    }
    for (;;) {
#pragma unroll
      for (int k = 0; k < kShSlots; k++) {
        const bool need = st[k] == 0;
        const unsigned nm = __ballot_sync(kFullMask, need);
        const int c = next_c + __popc(nm & lmask_lt());
        next_c += __popc(nm);
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int e = __shfl_sync(kFullMask, excl, lo + step);
          if (e <= c) lo += step;
        }
        const uint32_t m = __shfl_sync(kFullMask, pm, lo);
        const int ex = __shfl_sync(kFullMask, excl, lo);
        if (need && c < total) {
          const uint32_t bit = __fns(m, 0, c - ex + 1);
          r[k] = (uint32_t)((tbase + lo) * 32 + (int)bit);
          b[k] = P.off[r[k]];
          d[k] = (uint32_t)(P.off[r[k] + 1] - b[k]);
          rounds[k] = 0;
          st[k] = d[k] ? 2 : 0;
        }
      }
      bool active = false;
#pragma unroll
      for (int k = 0; k < kShSlots; k++) active |= st[k] != 0;
      if (__ballot_sync(kFullMask, active) == 0) {
        if (next_c >= total) break;
        continue;
      }
      uint32_t u[kShSlots][4];
#pragma unroll
      for (int k = 0; k < kShSlots; k++)
#pragma unroll
        for (int j = 0; j < 4; j++) u[k][j] = (st[k] && d[k] > (uint32_t)j) ? __ldg(P.nb + b[k] + j) : kNoVertex;
#pragma unroll
      for (int k = 0; k < kShSlots; k++) {
        if (!st[k]) continue;
        bool hit = false;
        uint32_t par = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          if (!hit && u[k][j] != kNoVertex && ((__ldg(front + (u[k][j] >> 5)) >> (u[k][j] & 31u)) & 1u)) {
            hit = true;
            par = u[k][j];
          }
        }
        if (hit) {
          P.parent[r[k]] = (int32_t)par;
          if (P.want_depth) P.depth[r[k]] = lvl + 1;
          atomicOr(&acc[(r[k] >> 5) - tbase], 1u << (r[k] & 31u));
          st[k] = 0;
        } else {
          const uint32_t tk = d[k] < 4u ? d[k] : 4u;
          b[k] += tk;
          d[k] -= tk;
          if (d[k] == 0) {
            st[k] = 0;
          } else if (++rounds[k] >= kShRounds) {
            const unsigned long long q = atomicAdd(&P.ctr[cLong], 1ull);
            if ((int64_t)q < P.long_cap) P.longq[q] = r[k];
            else atomicExch((unsigned*)&P.ctr[7], 1u);
            st[k] = 0;
          }
        }
      }
    }
    __syncwarp();
    if (lane < tw && w < w32) {
      const uint32_t nbits = acc[lane];
      next_slice[w] = nbits;
      if (nbits) P.visited[w] = vis | nbits;
      awake += __popc(nbits);
    }
    __syncwarp();
  }
  block_sum2(awake, 0, &P.ctr[cAwake], &P.ctr[cAwake]);
}

// Long in-lists deferred by k_sh_bu: one warp per vertex, ballot over 32
// neighbours, resuming after the kShRounds list rounds.
__global__ void __launch_bounds__(kSB) k_sh_bu_long(ShardParams P, const uint32_t* front, uint32_t* next_slice,
                                                    unsigned long long count, int lvl) {
  const int lane = threadIdx.x & 31;
  long long awake = 0;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = gw; i < (long long)count; i += nw) {
    const uint32_t r = P.longq[i];
    const int64_t le = P.off[r + 1];
    for (int64_t j = P.off[r] + 4 * kShRounds; j < le; j += 32) {
      const int64_t jj = j + lane;
      bool h = false;
      uint32_t u = 0;
      if (jj < le) {
        u = __ldg(P.nb + jj);
        h = (__ldg(front + (u >> 5)) >> (u & 31u)) & 1u;
      }
      const unsigned bal = __ballot_sync(kFullMask, h);
      if (bal) {
        const uint32_t hu = __shfl_sync(kFullMask, u, __ffs(bal) - 1);
        if (lane == 0) {
          P.parent[r] = (int32_t)hu;
          if (P.want_depth) P.depth[r] = lvl + 1;
          atomicOr(next_slice + (r >> 5), 1u << (r & 31u));
          atomicOr(P.visited + (r >> 5), 1u << (r & 31u));
          awake++;
        }
        break;
      }
    }
  }
  block_sum2(awake, 0, &P.ctr[cAwake], &P.ctr[cAwake]);
}

// Queue from the owned slice of the front (BitmapToQueue, bfs.hpp:99-113).
__global__ void __launch_bounds__(kSB) k_sh_b2q(ShardParams P, const uint32_t* slice) {
  // warp prefix sum of popcounts, one fetch-add per warp; entries in vertex order
  const long long w32 = (P.nloc + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; w0 < w32;
       w0 += (long long)gridDim.x * blockDim.x) {
    const long long w = w0 + lane;
    uint32_t word = w < w32 ? __ldcg(slice + w) : 0u;
    const int cnt = __popc(word);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(kFullMask, incl, 31);
    if (total == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&P.ctr[cTail], (unsigned long long)total);
    base = __shfl_sync(kFullMask, base, 0);
    unsigned long long q = base + incl - cnt;
    while (word) {
      const int bp = __ffs(word) - 1;
      word &= word - 1;
      if ((int64_t)q < P.nloc + 1) P.queue[q] = (uint32_t)(P.lo + w * 32 + bp);
      else atomicExch((unsigned*)&P.ctr[7], 1u);
      q++;
    }
  }
}

// m_cc contribution: (reached, sum of degrees of reached owned vertices).
__global__ void k_sh_count(ShardParams P, unsigned long long* out) {
  long long r = 0, d = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P.nloc;
       i += (long long)gridDim.x * blockDim.x)
    if (P.parent[i] >= 0) {
      r++;
      d += P.off[i + 1] - P.off[i];
    }
  block_sum2(r, d, out, out + 1);
}

int grid_of(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (work + kSB - 1) / kSB;
  return (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * 4));
}

}  // namespace
}  // namespace gk

// ---------------------------------------------------------------- C ABI
struct gk_shard {
  int device = 0;
  int rank = 0, nranks = 1;
  int64_t n = 0, lo = 0, hi = 0, nloc = 0, block = 0, m = 0;
  int64_t* off = nullptr;
  uint32_t* nb = nullptr;
  int32_t* parent = nullptr;
  int32_t* depth = nullptr;
  uint32_t* visited = nullptr;
  uint32_t* sent = nullptr;
  uint32_t* queue = nullptr;
  uint64_t* pairs = nullptr;
  int64_t pair_cap = 0;
  gk::Chunk* chunks = nullptr;
  int64_t chunk_cap = 0;
  unsigned long long* ctr = nullptr;  // device counters
  unsigned long long* acc = nullptr;
  cudaStream_t stream = nullptr;  // caller's stream (e.g. torch's current stream)
  int want_depth = 0;
  int encode = 1;
  int big = 0;                  // the current top-down step is a large one
  uint32_t* next = nullptr;     // owned next bitmap for large top-down steps
  uint32_t* dead = nullptr;     // owned never-reachable bitmap (built once)
  long long launches = 0;  // kernels launched on this shard (telemetry)
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

gk::ShardParams params(const gk_shard* s) {
  gk::ShardParams p{};
  p.n = s->n;
  p.lo = s->lo;
  p.hi = s->hi;
  p.nloc = s->nloc;
  p.block = s->block;
  p.rank = s->rank;
  p.nranks = s->nranks;
  p.off = s->off;
  p.nb = s->nb;
  p.parent = s->parent;
  p.depth = s->depth;
  p.visited = s->visited;
  p.sent = s->sent;
  p.queue = s->queue;
  p.pairs = s->pairs;
  p.pair_cap = s->pair_cap;
  p.chunks = s->chunks;
  p.chunk_cap = s->chunk_cap;
  p.ctr = s->ctr;
  p.want_depth = s->want_depth;
  p.encode = s->encode;
  p.big = s->big;
  p.next = s->next;
  p.dead = s->dead;
  p.longq = reinterpret_cast<uint32_t*>(s->pairs);
  p.long_cap = 2 * s->pair_cap;
  return p;
}

gk_status shard_alloc(gk_shard* s) {
  {  // the owned rows must be a valid CSR over global neighbour ids
    bool off_ok = true, ids_ok = true;
    SCK(gk::validate_csr(s->off, s->nb, s->nloc, s->m, s->n, &off_ok, &ids_ok, nullptr, nullptr), "validate shard CSR");
    if (!off_ok) return shard_fail(GK_ERR_INVALID, "invalid shard: offsets not monotone from 0 to m");
    if (!ids_ok) return shard_fail(GK_ERR_INVALID, "invalid shard: neighbour id out of range");
  }
  const int64_t wl = (s->nloc + 31) / 32 + 4, wg = (s->n + 31) / 32 + 4;
  SCK(cudaMalloc(&s->parent, sizeof(int32_t) * std::max<int64_t>(s->nloc, 1)), "alloc parent");
  SCK(cudaMalloc(&s->depth, sizeof(int32_t) * std::max<int64_t>(s->nloc, 1)), "alloc depth");
  SCK(cudaMalloc(&s->visited, sizeof(uint32_t) * wl), "alloc visited");
  SCK(cudaMalloc(&s->sent, sizeof(uint32_t) * wg), "alloc sent");
  SCK(cudaMalloc(&s->queue, sizeof(uint32_t) * (s->nloc + 2)), "alloc queue");
  s->pair_cap = std::max<int64_t>(s->m, 1024);
  SCK(cudaMalloc(&s->pairs, sizeof(uint64_t) * s->pair_cap), "alloc pairs");
  s->chunk_cap = 2 * (s->m / 1024) + 64;
  SCK(cudaMalloc(&s->chunks, sizeof(gk::Chunk) * s->chunk_cap), "alloc chunks");
  SCK(cudaMalloc(&s->ctr, sizeof(unsigned long long) * (gk::cDest + s->nranks + 8)), "alloc counters");
  SCK(cudaMalloc(&s->acc, sizeof(unsigned long long) * 4), "alloc acc");
  SCK(cudaMalloc(&s->next, sizeof(uint32_t) * wl), "alloc next");
  SCK(cudaMalloc(&s->dead, sizeof(uint32_t) * wl), "alloc dead");
  // graph layout, once: never-reachable owned vertices
  int64_t nlive = 0;
  SCK(gk::dead_bitmap(s->off, s->nloc, s->dead, &nlive, nullptr), "dead bitmap");
  return GK_OK;
}

void shard_free(gk_shard* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  for (void* p : {(void*)s->off, (void*)s->nb, (void*)s->parent, (void*)s->depth, (void*)s->visited,
                  (void*)s->sent, (void*)s->queue, (void*)s->pairs, (void*)s->chunks,
                  (void*)s->ctr, (void*)s->acc, (void*)s->next, (void*)s->dead})
    cudaFree(p);
  delete s;
}

int64_t block_of(int64_t n, int nranks) {
  int64_t b = (n + nranks - 1) / nranks;
  return (b + 31) / 32 * 32;
}

gk_status read_ctr(gk_shard* s, unsigned long long* h, int count) {
  SCK(cudaMemcpyAsync(h, s->ctr, sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost, s->stream), "D2H");
  SCK(cudaStreamSynchronize(s->stream), "sync");
  if (h[7]) return shard_fail(GK_ERR_CUDA, "shard buffer overflow");
  return GK_OK;
}
}  // namespace

extern "C" {

GK_API const char* gk_shard_last_error(void) { return g_shard_err.c_str(); }

GK_API gk_status gk_shard_generate(int kind, int scale, int degree, uint64_t seed, int permute, int rank,
                                   int nranks, int device, gk_shard** out) {
  if (!out || nranks < 1 || nranks > gk::kMaxRanksSmem || rank < 0 || rank >= nranks)
    return shard_fail(GK_ERR_INVALID, "bad shard spec");
  if (kind != 0 && kind != 1) return shard_fail(GK_ERR_INVALID, "generator kind must be 0 or 1");
  if (scale < 5 || scale > 31) return shard_fail(GK_ERR_INVALID, "sharded generator scale must be in [5, 31]");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return shard_fail(GK_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
  SCK(cudaSetDevice(device), "cudaSetDevice");
  auto* s = new gk_shard;
  s->device = device;
  s->rank = rank;
  s->nranks = nranks;
  s->n = int64_t{1} << scale;
  s->block = block_of(s->n, nranks);
  s->lo = std::min<int64_t>(s->n, rank * s->block);
  s->hi = std::min<int64_t>(s->n, s->lo + s->block);
  s->nloc = s->hi - s->lo;
  gk::DevCsr csr;
  std::string err;
  cudaError_t e = gk::build_generated(kind, scale, degree, seed, permute, s->lo, s->hi, &csr, &err);
  if (e != cudaSuccess) {
    delete s;
    return shard_fail(GK_ERR_CUDA, err.empty() ? cudaGetErrorString(e) : err);
  }
  s->off = csr.off;
  s->nb = csr.nb;
  s->m = csr.m;
  gk_status st = shard_alloc(s);
  if (st != GK_OK) {
    shard_free(s);
    return st;
  }
  *out = s;
  return GK_OK;
}

GK_API gk_status gk_shard_upload(int64_t n, int rank, int nranks, const int64_t* local_offsets,
                                 const uint32_t* neighbors, int device, gk_shard** out) {
  if (!out || !local_offsets || nranks < 1 || nranks > gk::kMaxRanksSmem || rank < 0 || rank >= nranks || n < 1)
    return shard_fail(GK_ERR_INVALID, "bad shard spec");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return shard_fail(GK_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
  SCK(cudaSetDevice(device), "cudaSetDevice");
  auto* s = new gk_shard;
  s->device = device;
  s->rank = rank;
  s->nranks = nranks;
  s->n = n;
  s->block = block_of(n, nranks);
  s->lo = std::min<int64_t>(n, rank * s->block);
  s->hi = std::min<int64_t>(n, s->lo + s->block);
  s->nloc = s->hi - s->lo;
  s->m = local_offsets[s->nloc];
  cudaError_t e;
  if ((e = cudaMalloc(&s->off, sizeof(int64_t) * (s->nloc + 3))) ||
      (e = cudaMalloc(&s->nb, sizeof(uint32_t) * std::max<int64_t>(s->m, 1) + gk::kNbPad)) ||
      (e = cudaMemcpy(s->off, local_offsets, sizeof(int64_t) * (s->nloc + 1), cudaMemcpyHostToDevice)) ||
      (s->m && (e = cudaMemcpy(s->nb, neighbors, sizeof(uint32_t) * s->m, cudaMemcpyHostToDevice)))) {
    shard_free(s);
    return shard_fail(GK_ERR_CUDA, cudaGetErrorString(e));
  }
  gk_status st = shard_alloc(s);
  if (st != GK_OK) {
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

GK_API gk_status gk_shard_set_stream(gk_shard* s, void* stream) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  s->stream = (cudaStream_t)stream;
  return GK_OK;
}

GK_API gk_status gk_shard_degree(const gk_shard* s, uint32_t v, int64_t* deg) {
  if (!s || !deg || (int64_t)v < s->lo || (int64_t)v >= s->hi) return shard_fail(GK_ERR_INVALID, "vertex not owned");
  int64_t o[2];
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  SCK(cudaMemcpy(o, s->off + (v - s->lo), sizeof(o), cudaMemcpyDeviceToHost), "D2H");
  *deg = o[1] - o[0];
  return GK_OK;
}

// Start a traversal: reset owned state; the owner of src claims it.
GK_API gk_status gk_shard_begin(gk_shard* s, uint32_t src, int32_t strategy, int32_t want_depth) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  if ((int64_t)src >= s->n) return shard_fail(GK_ERR_SOURCE_RANGE, "bfs source out of range");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  s->want_depth = want_depth ? 1 : 0;
  s->encode = strategy != GK_BFS_TOP_DOWN_RESCAN;
  gk::ShardParams p = params(s);
  SCK(cudaMemsetAsync(s->ctr, 0, sizeof(unsigned long long) * (gk::cDest + s->nranks + 8), s->stream), "memset");
  s->launches++;
  gk::k_sh_init<<<gk::grid_of(s->nloc), gk::kSB, 0, s->stream>>>(p);
  if ((int64_t)src >= s->lo && (int64_t)src < s->hi) {
    s->launches++;
    gk::k_sh_set_source<<<1, 1, 0, s->stream>>>(p, src);
  }
  SCK(cudaGetLastError(), "begin");
  return GK_OK;
}

// Top-down expansion of the owned window [qs, qe).  Outputs (host):
//   local[0] = claims made in place, local[1] = their scout,
//   dest_counts[r] = pairs for rank r, laid out by rank in *pairs_dev.
GK_API gk_status gk_shard_td_expand(gk_shard* s, uint64_t qs, uint64_t qe, int32_t lvl, int32_t dedup,
                                    int64_t* local, int64_t* dest_counts, uint64_t* pairs_out_dev,
                                    int64_t pairs_cap) {
  if (!s || !local || !dest_counts || (!pairs_out_dev && s->nranks > 1))
    return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  gk::ShardParams p = params(s);
  p.dedup = dedup ? 1 : 0;
  p.pairs_out = pairs_out_dev;
  const int P = s->nranks;
  SCK(cudaMemsetAsync(s->ctr + gk::cPairs, 0, sizeof(unsigned long long), s->stream), "memset");
  SCK(cudaMemsetAsync(s->ctr + gk::cScout, 0, sizeof(unsigned long long) * 2, s->stream), "memset");
  SCK(cudaMemsetAsync(s->ctr + gk::cChunks, 0, sizeof(unsigned long long), s->stream), "memset");
  SCK(cudaMemsetAsync(s->ctr + gk::cDest, 0, sizeof(unsigned long long) * P, s->stream), "memset");
  // one rank has no remote targets: no sent-bitmap to clear or probe
  p.dedup = (dedup && s->nranks > 1) ? 1 : 0;
  if (p.dedup) SCK(cudaMemsetAsync(s->sent, 0, sizeof(uint32_t) * ((s->n + 31) / 32), s->stream), "memset");
  // large steps (the orchestrator's dedup threshold = the persistent
  // kernel's "big" threshold): owned claims go to next := visited
  s->big = dedup ? 1 : 0;
  p.big = s->big;
  if (s->big) {
    s->launches++;
    gk::k_sh_copy_words<<<gk::grid_of((s->nloc + 31) / 32), gk::kSB, 0, s->stream>>>(s->visited, s->next,
                                                                                  (s->nloc + 31) / 32);
  }
  s->launches++;
  gk::k_sh_td_light<<<gk::grid_of((int64_t)(qe - qs)), gk::kSB, 0, s->stream>>>(p, qs, qe, lvl);
  SCK(cudaGetLastError(), "td_light");
  unsigned long long h[gk::cDest + 64];
  gk_status st = read_ctr(s, h, gk::cDest);
  if (st != GK_OK) return st;
  if (h[gk::cChunks]) {
    s->launches++;
    gk::k_sh_td_heavy<<<gk::grid_of((int64_t)h[gk::cChunks] * 32), gk::kSB, 0, s->stream>>>(p, h[gk::cChunks], lvl);
    SCK(cudaGetLastError(), "td_heavy");
    st = read_ctr(s, h, gk::cDest);
    if (st != GK_OK) return st;
  }
  const unsigned long long npairs = h[gk::cPairs];
  if ((int64_t)npairs > pairs_cap) return shard_fail(GK_ERR_INVALID, "pairs buffer too small");
  std::vector<unsigned long long> cursor(P, 0);
  if (npairs) {
    s->launches += 2;
    gk::k_sh_count_dest<<<gk::grid_of((int64_t)npairs), gk::kSB, 0, s->stream>>>(p, npairs);
    SCK(cudaGetLastError(), "count_dest");
    st = read_ctr(s, h, gk::cDest + P);
    if (st != GK_OK) return st;
    unsigned long long run = 0;
    for (int r = 0; r < P; r++) {
      cursor[r] = run;
      run += h[gk::cDest + r];
    }
    SCK(cudaMemcpyAsync(s->ctr + gk::cDest, cursor.data(), sizeof(unsigned long long) * P, cudaMemcpyHostToDevice,
                        s->stream),
        "H2D");
    gk::k_sh_scatter_dest<<<gk::grid_of((int64_t)npairs), gk::kSB, 0, s->stream>>>(p, npairs, s->ctr + gk::cDest);
    SCK(cudaGetLastError(), "scatter_dest");
  } else {
    for (int r = 0; r < P; r++) h[gk::cDest + r] = 0;
  }
  for (int r = 0; r < P; r++) dest_counts[r] = npairs ? (int64_t)h[gk::cDest + r] : 0;
  local[0] = (int64_t)h[gk::cClaims];
  local[1] = (int64_t)h[gk::cScout];
  SCK(cudaStreamSynchronize(s->stream), "td_expand");
  return GK_OK;
}

// Claims from received pairs (device array, npairs entries).  out[0] =
// claims, out[1] = scout; new queue entries are appended after the local ones.
GK_API gk_status gk_shard_td_apply(gk_shard* s, const uint64_t* pairs_in, int64_t npairs, int32_t lvl,
                                   int64_t* out) {
  if (!s || !out) return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  gk::ShardParams p = params(s);
  SCK(cudaMemsetAsync(s->ctr + gk::cScout, 0, sizeof(unsigned long long) * 2, s->stream), "memset");
  if (npairs > 0) {
    s->launches++;
    gk::k_sh_td_apply<<<gk::grid_of(npairs), gk::kSB, 0, s->stream>>>(p, pairs_in, (unsigned long long)npairs, lvl);
    SCK(cudaGetLastError(), "td_apply");
  }
  if (s->big) {  // claim sweep: fold, queue, scout for the whole step
    s->launches++;
    gk::k_sh_sweep<<<gk::grid_of(s->nloc / 32), gk::kSB, 0, s->stream>>>(p, lvl);
    SCK(cudaGetLastError(), "sweep");
    s->big = 0;
  }
  unsigned long long h[gk::cDest];
  gk_status st = read_ctr(s, h, gk::cDest);
  if (st != GK_OK) return st;
  out[0] = (int64_t)h[gk::cClaims];
  out[1] = (int64_t)h[gk::cScout];
  return GK_OK;
}

GK_API gk_status gk_shard_tail(gk_shard* s, uint64_t* tail) {
  if (!s || !tail) return shard_fail(GK_ERR_INVALID, "null argument");
  unsigned long long h[gk::cDest];
  gk_status st = read_ctr(s, h, gk::cDest);
  if (st != GK_OK) return st;
  *tail = h[gk::cTail];
  return GK_OK;
}

// Sum of degrees of the owned queue window (kTopDownRescan, bfs.hpp:161-167).
GK_API gk_status gk_shard_rescan(gk_shard* s, uint64_t qs, uint64_t qe, int64_t* total) {
  if (!s || !total) return shard_fail(GK_ERR_INVALID, "null argument");
  std::vector<uint32_t> q(qe - qs);
  std::vector<int64_t> off(s->nloc + 1);
  SCK(cudaStreamSynchronize(s->stream), "sync");
  if (qe > qs) SCK(cudaMemcpy(q.data(), s->queue + qs, sizeof(uint32_t) * (qe - qs), cudaMemcpyDeviceToHost), "D2H");
  SCK(cudaMemcpy(off.data(), s->off, sizeof(int64_t) * (s->nloc + 1), cudaMemcpyDeviceToHost), "D2H");
  int64_t t = 0;
  for (uint32_t v : q) t += off[v - s->lo + 1] - off[v - s->lo];
  *total = t;
  return GK_OK;
}

// Owned slice (words) of the front bitmap from the queue window [qs, qe).
GK_API gk_status gk_shard_q2b(gk_shard* s, uint64_t qs, uint64_t qe, uint32_t* slice_dev) {
  if (!s || !slice_dev) return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  gk::ShardParams p = params(s);
  SCK(cudaMemsetAsync(slice_dev, 0, sizeof(uint32_t) * (s->block / 32), s->stream), "memset");
  if (qe > qs) s->launches++;
  if (qe > qs) gk::k_sh_q2b<<<gk::grid_of((int64_t)(qe - qs)), gk::kSB, 0, s->stream>>>(p, qs, qe, slice_dev);
  SCK(cudaGetLastError(), "q2b");
  return GK_OK;
}

// Bottom-up step: front_dev = replicated n-bit bitmap (block*nranks bits);
// writes the owned slice of next; *awake = vertices found here.
GK_API gk_status gk_shard_bu(gk_shard* s, const uint32_t* front_dev, uint32_t* next_slice_dev, int32_t lvl,
                             int64_t* awake) {
  if (!s || !front_dev || !next_slice_dev || !awake) return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  gk::ShardParams p = params(s);
  SCK(cudaMemsetAsync(s->ctr + gk::cAwake, 0, sizeof(unsigned long long), s->stream), "memset");
  SCK(cudaMemsetAsync(next_slice_dev, 0, sizeof(uint32_t) * (s->block / 32), s->stream), "memset");
  SCK(cudaMemsetAsync(s->ctr + gk::cLong, 0, sizeof(unsigned long long), s->stream), "memset");
  s->launches++;
  gk::k_sh_bu<<<gk::grid_of(s->nloc), gk::kSB, 0, s->stream>>>(p, front_dev, next_slice_dev, lvl);
  SCK(cudaGetLastError(), "bu");
  unsigned long long h[gk::cDest];
  gk_status st = read_ctr(s, h, gk::cDest);
  if (st != GK_OK) return st;
  if (h[gk::cLong]) {
    s->launches++;
    gk::k_sh_bu_long<<<gk::grid_of((int64_t)h[gk::cLong] * 32), gk::kSB, 0, s->stream>>>(p, front_dev, next_slice_dev,
                                                                                       h[gk::cLong], lvl);
    SCK(cudaGetLastError(), "bu_long");
    st = read_ctr(s, h, gk::cDest);
    if (st != GK_OK) return st;
  }
  *awake = (int64_t)h[gk::cAwake];
  return GK_OK;
}

// Queue entries from the owned slice of the front (appended at the tail).
GK_API gk_status gk_shard_b2q(gk_shard* s, const uint32_t* slice_dev) {
  if (!s || !slice_dev) return shard_fail(GK_ERR_INVALID, "null argument");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  gk::ShardParams p = params(s);
  s->launches++;
  gk::k_sh_b2q<<<gk::grid_of((s->nloc + 31) / 32), gk::kSB, 0, s->stream>>>(p, slice_dev);
  SCK(cudaGetLastError(), "b2q");
  return GK_OK;
}

// Owned results: parent (and depth when requested) for [lo, hi), plus
// counts[0] = reached, counts[1] = sum of degrees of reached owned vertices.
GK_API gk_status gk_shard_result(gk_shard* s, int32_t* parent_out, int32_t* depth_out, int64_t* counts) {
  if (!s) return shard_fail(GK_ERR_INVALID, "null shard");
  SCK(cudaSetDevice(s->device), "cudaSetDevice");
  if (counts) {
    gk::ShardParams p = params(s);
    SCK(cudaMemsetAsync(s->acc, 0, sizeof(unsigned long long) * 2, s->stream), "memset");
    s->launches++;
    gk::k_sh_count<<<gk::grid_of(s->nloc), gk::kSB, 0, s->stream>>>(p, s->acc);
    unsigned long long two[2];
    SCK(cudaMemcpyAsync(two, s->acc, sizeof(two), cudaMemcpyDeviceToHost, s->stream), "D2H");
    SCK(cudaStreamSynchronize(s->stream), "sync");
    counts[0] = (int64_t)two[0];
    counts[1] = (int64_t)two[1];
  }
  if (parent_out && s->nloc)
    SCK(cudaMemcpyAsync(parent_out, s->parent, sizeof(int32_t) * s->nloc, cudaMemcpyDeviceToHost, s->stream), "D2H");
  if (depth_out && s->nloc && s->want_depth)
    SCK(cudaMemcpyAsync(depth_out, s->depth, sizeof(int32_t) * s->nloc, cudaMemcpyDeviceToHost, s->stream), "D2H");
  SCK(cudaStreamSynchronize(s->stream), "sync");
  return GK_OK;
}

}  // extern "C"
