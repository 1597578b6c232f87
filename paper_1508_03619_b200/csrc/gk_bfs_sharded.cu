// gk_bfs_sharded.cu -- the 1D-partitioned direction-optimizing BFS of
// SURVEY.md §8(e) as ONE persistent kernel per rank: the level loop of
// bfs.hpp:139-169 runs on the device, ranks exchange bitmap slices through
// peer memory (NVLink P2P stores / loads) and meet at a cross-rank barrier
// that also reduces the heuristic's counters, so no host round trip sits
// between levels.
//
// Partition: rank r owns vertices [lo, hi) and their CSR rows (undirected:
// in = out); every rank holds full-n replicated bitmaps (visited, the
// front/next pair, claims) and the graph's dead bitmap; parents and depths
// cover the owned range.
//
// Per bottom-up step (bfs.hpp:47-66): each rank sweeps its owned pending
// vertices against its replicated front (the single-device bu_step /
// bu_long on the owned words), then writes its owned slice of next into
// every peer's next (all-gather by P2P stores).
// Per top-down step (bfs.hpp:68-91): each rank expands its owned frontier
// vertices (the single-device tile / heavy-chunk expansion) setting bits in
// its own full-n claims bitmap and storing the parent into the target
// owner's parent array (a fire-and-forget NVLink store when remote; racing
// claimers store valid parents, as the single-device claims do); after the
// barrier each owner ORs the peers' claims over its own words (P2P loads: a
// reduce-scatter of bitmaps), keeps the unvisited ones, sums their degrees
// (scout) and all-gathers the slice.
// Counters (scout, awake, claims) are reduced at every cross-rank barrier,
// so every rank takes the reference's direction decisions from the same
// totals and the schedule equals the single-device one.
//
// Launch modes: one launch per device (multi-device; the cross-rank barrier
// and counters live in rank 0's XCtrl, mapped by the others), or all ranks
// in ONE cooperative launch on one device, cpr CTAs per rank (emulation:
// B200_PROFILING.md forbids ranks that wait on one another as separate
// launches on one GPU).  Both run the same phases; only the barrier differs.
// NVLink bytes received per rank and level: (P-1)/P * n/8 per step (the
// all-gather) plus (P-1)/P * n/8 per top-down step (the claims reduce).
#include <algorithm>

#define GK_SHARDED_STEPS 1
#include "gk_bfs_steps.cuh"

namespace gk {
namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ void rank_params(BfsParams& Q, const BfsParams& P0, const ShardTab& T, int r) {
  Q = P0;
  const ShardView& v = T.v[r];
  Q.out_off = Q.in_off = v.off;
  Q.off32 = v.off32;  // the rank's rows in compact form (shifted like off), or null
  Q.off_hi[0] = v.off_hi;
  Q.out_nb = Q.in_nb = v.nb;
  Q.parent = v.parent;
  Q.depth = v.depth;
  Q.queue = v.queue;
  Q.chunks = v.chunks;
  Q.chunk_cap = v.chunk_cap;
  Q.visited = v.bm[0];
  Q.bm0 = v.bm[1];
  Q.bm1 = v.bm[2];
  Q.dead = v.dead;
  Q.w_lo = v.lo >> 5;  // lo is a multiple of 1024 unless the rank is empty (lo = hi = n)
  Q.w_hi = v.hi > v.lo ? (v.hi + 31) >> 5 : Q.w_lo;
  Q.cpr = T.emulated ? P0.cpr : 0;
  Q.rslot = T.emulated ? r + 1 : 0;
  Q.sharded = 1;
  Q.shard_block = T.block;
  Q.shard_recip = (uint32_t)(((1ull << 32) + (unsigned long long)T.block - 1) / (unsigned long long)T.block);
  for (int q = 0; q < kMaxRanks; q++) Q.shard_parent[q] = q < T.nranks ? T.v[q].parent : nullptr;
  Q.front_in_smem = 0;
  Q.own_list = v.own_list;  // owned-range hub geometry (own_r, own_span_w, ...) is the same for every rank
  Q.own_stage = v.own_stage;
  Q.own_cap = v.own_cap;
}

// Barrier across all ranks of the traversal.  Emulation: the launch's grid
// barrier (all ranks share one Ctrl, so its totals are traversal-wide).
// Multi-device: a grid barrier of this rank, then its CTA 0 adds the rank's
// totals into rank 0's XCtrl, arrives (release, system scope) and waits for
// every rank (acquire), copies the totals back, and a second grid barrier
// releases the rank's CTAs with them in s.snap.
__device__ bool xsync(const BfsParams& Q, const ShardTab& T, SmemT& s, unsigned& ph, unsigned& xph,
                      unsigned char tag) {
  if (T.emulated || (T.nranks == 1 && !T.force_x)) return grid_sync(Q, s, ph, tag);
  __threadfence_system();  // this phase's peer stores, before the arrival
  if (!grid_sync(Q, s, ph, tag)) return false;
  unsigned long long keep[kSlots];
#pragma unroll
  for (int i = 0; i < kSlots; i++) keep[i] = s.snap[i];
  if (cta_id(Q) == 0 && threadIdx.x == 0) {
    XCtrl* X = T.x;
    const unsigned long long xi = T.xbase + xph;  // cross-rank barrier index since the group was wired
    const unsigned set = (unsigned)(xi & 3);
#pragma unroll
    for (int k = 0; k < kSlots; k++)
      if (global_slot(k) && keep[k]) atomicAdd_system(&X->cnt[set][k], keep[k]);
    red_release_sys(&X->bar, 1ull);
    const unsigned long long target = (xi + 1) * (unsigned long long)T.nranks;
    unsigned long long t0 = 0;
    unsigned spins = 0;
    while (ld_acquire_sys(&X->bar) < target) {
      if ((++spins & 255u) == 0) {
        if (*reinterpret_cast<volatile int*>(&X->error)) {
          atomicExch(&Q.ctrl->error, 2);
          break;
        }
        const unsigned long long now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > Q.timeout_ns) {
          atomicExch_system(&X->error, 2);
          atomicExch(&Q.ctrl->error, 2);
          break;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kSlots; k++)
      Q.ctrl->xsnap[k] = global_slot(k) ? *reinterpret_cast<volatile unsigned long long*>(&X->cnt[set][k]) : 0ull;
    if (T.rank == 0) {  // recycle the set two barriers ahead (its last readers are past barrier xph)
#pragma unroll
      for (int k = 0; k < kSlots; k++) X->cnt[(xi + 2) & 3][k] = 0;
    }
  }
  if (!grid_sync(Q, s, ph, tag)) return false;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kSlots; i++) s.snap[i] = global_slot(i) ? __ldcg(&Q.ctrl->xsnap[i]) : keep[i];
    s.ok = *reinterpret_cast<volatile int*>(&Q.ctrl->error) == 0;
  }
  __syncthreads();
  xph++;
  return s.ok != 0;
}

// The owned words of this rank's bitmap `role` (1/2: the front/next pair)
// written into the same bitmap of every peer (all-gather by P2P stores).
__device__ void broadcast_owned(const BfsParams& Q, const ShardTab& T, int r, int role, long long gtid,
                                long long gthreads) {
  if (T.nranks == 1) return;
  const uint32_t* mine = T.v[r].bm[role];
  const long long a = Q.w_lo, b = Q.w_hi;
  const long long b4 = a + ((b - a) & ~3ll);  // w_lo is a multiple of 32 words: 16-byte aligned
  for (long long w = a + 4 * gtid; w < b4; w += 4 * gthreads) {
    const uint4 x = __ldcg(reinterpret_cast<const uint4*>(mine + w));
    for (int q = 0; q < T.nranks; q++)
      if (q != r) __stcg(reinterpret_cast<uint4*>(T.v[q].bm[role] + w), x);
  }
  for (long long w = b4 + gtid; w < b; w += gthreads) {
    const uint32_t x = __ldcg(mine + w);
    for (int q = 0; q < T.nranks; q++)
      if (q != r) __stcg(T.v[q].bm[role] + w, x);
  }
}

// Top-down merge over the owned words (a warp per 32 words, lane = word):
// claims = OR over every rank's claims bitmap & ~visited; they become the
// owned slice of next and are folded into visited; their count, degree sum
// (scout = sum of max(deg, 1), bfs.hpp:83 with bfs.hpp:130's encoding) and
// depths are recorded.  (Their parents were stored by the claimers.)
__device__ void merge_claims(const BfsParams& Q, const ShardTab& T, int r, uint32_t* next, int lvl,
                             long long& scout, long long& count) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)cta_id(Q) * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)cta_count(Q) * kBlock) >> 5;
  const uint32_t* own_claims = T.v[r].bm[3];
  for (long long w0 = Q.w_lo + gw * 32; w0 < Q.w_hi; w0 += nw * 32) {
    const long long w = w0 + lane;
    uint32_t cl = 0;
    if (w < Q.w_hi) {
      uint32_t c = ld_bits(own_claims + w);
      for (int q = 0; q < T.nranks; q++)
        if (q != r) c |= __ldcg(T.v[q].bm[3] + w);
      const uint32_t vis = ld_bits(Q.visited + w);
      cl = c & ~vis;
      next[w] = cl;
      if (cl) Q.visited[w] = vis | cl;
    }
    count += __popc(cl);
    scout += claim_degrees(Q, w0, cl);  // owned rows
    if (Q.want_depth)
      for (uint32_t m = cl; m; m &= m - 1) Q.depth[w * 32 + (__ffs(m) - 1)] = lvl + 1;
  }
}

__global__ void __launch_bounds__(kBlock, 2) bfs_sharded(BfsParams P0, ShardTab T) {
  extern __shared__ uint4 dyn_smem[];
  __shared__ SmemT s;
  __shared__ BfsParams Q;  // this CTA's rank view (read through shared memory by every phase)
  const int r = T.emulated ? (int)(blockIdx.x / P0.cpr) : T.rank;
  if (threadIdx.x == 0) rank_params(Q, P0, T, r);
  __syncthreads();
  const ShardView& me = T.v[r];
  unsigned ph = 0, xph = 0;
  const long long gtid = (long long)cta_id(Q) * kBlock + threadIdx.x;
  const long long gthreads = (long long)cta_count(Q) * kBlock;
  const uint32_t src = Q.src;
  const bool owner = (int64_t)src >= me.lo && (int64_t)src < me.hi;
  uint32_t* const vis = me.bm[0];
  uint32_t* const claims = me.bm[3];
  uint32_t* const wsm = reinterpret_cast<uint32_t*>(dyn_smem);
  if (blockIdx.x == 0 && threadIdx.x == 0) Q.ctrl->ts[0] = globaltimer();

  // ---- init (timed; bfs.hpp:126-138): owned parents := -1, replicated
  // visited := the dead set, front := {} ----
  for (long long i = me.lo + gtid; i < me.hi; i += gthreads) {
    Q.parent[i] = -1;
    if (Q.want_depth) Q.depth[i] = -1;
  }
  for (long long w = gtid; w < Q.w32; w += gthreads) {
    vis[w] = __ldg(Q.dead + w);
    me.bm[1][w] = 0u;
  }
  if (!xsync(Q, T, s, ph, xph, kTagInit)) return;
  if (cta_id(Q) == 0 && threadIdx.x == 0) {  // bfs.hpp:132-136 on every replica; scout = deg(src)
    vis[src >> 5] |= 1u << (src & 31u);
    me.bm[1][src >> 5] |= 1u << (src & 31u);
    if (owner) {
      Q.parent[src] = (int32_t)src;
      if (Q.want_depth) Q.depth[src] = 0;
      atomicAdd(&Q.ctrl->cnt[ph & 3][kSum], (unsigned long long)(Q.out_off[src + 1] - Q.out_off[src]));
    }
  }
  if (!xsync(Q, T, s, ph, xph, kTagInit)) return;

  const bool encode = Q.strategy != GK_BFS_TOP_DOWN_RESCAN;
  long long scout = (long long)s.snap[kSum];  // bfs.hpp:140
  long long etc = T.m_total;                  // bfs.hpp:139
  long long gfront = 1, reached = 1, nsteps = 0, dummy = 0;
  unsigned long long qtail = 0;  // this rank's queue (owned frontier windows)
  int lvl = 0, cur = 0, qcnt = 0;
  const long long nwarps = gthreads >> 5;
  int bu_tw_log = Q.bu_tw_log_max;
  while (bu_tw_log > 0 && ((Q.w_hi - Q.w_lo + (1 << bu_tw_log) - 1) >> bu_tw_log) < nwarps) bu_tw_log--;

  while (gfront > 0) {
    if (Q.strategy == GK_BFS_DIRECTION_OPTIMIZING && scout > etc / Q.alpha) {  // bfs.hpp:143-156
      long long awake = gfront, old_awake;  // bfs.hpp:146
      do {
        old_awake = awake;
        uint32_t* frontg = me.bm[1 + cur];
        uint32_t* nextg = me.bm[2 - cur];
        // peers' claims of the last level join this replica's visited words
        for (long long w = gtid; w < Q.w32; w += gthreads)
          if (w < Q.w_lo || w >= Q.w_hi) vis[w] |= __ldcg(frontg + w);
        long long acc = 0;
        bu_step<false>(Q, s, ph, frontg, nextg, lvl, 0, bu_tw_log, acc, wsm);
        block_add(acc, &Q.ctrl->cnt[ph & 3][kSum], s);
        if (!xsync(Q, T, s, ph, xph, kTagBU)) return;
        awake = (long long)s.snap[kSum];
        if (s.snap[kWork]) {  // some rank deferred long lists
          const unsigned long long nlong = s.snap[kLongCount];
          acc = 0;
          bu_long<false>(Q, frontg, nextg, Q.queue, nlong, lvl, acc, dummy);
          block_add(acc, &Q.ctrl->cnt[ph & 3][kSum], s);
          if (!xsync(Q, T, s, ph, xph, kTagLong)) return;
          awake += (long long)s.snap[kSum];
        }
        if (T.nranks > 1) {
          broadcast_owned(Q, T, r, 2 - cur, gtid, gthreads);  // all-gather of next
          if (!xsync(Q, T, s, ph, xph, kTagZero)) return;
        }
        reached += awake;
        log_step(Q, nsteps++, 'B', old_awake, awake, etc);
        lvl++;
        cur ^= 1;
      } while (awake >= old_awake || awake > Q.n / Q.beta);  // bfs.hpp:154
      scout = 1;  // bfs.hpp:156
      gfront = awake;
    } else {
      etc -= scout;  // bfs.hpp:158
      const long long fsize = gfront;
      uint32_t* frontg = me.bm[1 + cur];
      uint32_t* nextg = me.bm[2 - cur];
      // Z: the last level joins visited; claims := visited; owned frontier -> queue
      for (long long w = gtid; w < Q.w32; w += gthreads) {
        uint32_t v = __ldcg(vis + w);
        if (w < Q.w_lo || w >= Q.w_hi) {
          v |= __ldcg(frontg + w);
          vis[w] = v;
        }
        claims[w] = v;
      }
      b2q(Q, qapp(Q, ph, qtail), frontg);
      if (!xsync(Q, T, s, ph, xph, kTagB2Q)) return;
      const unsigned long long qs = qtail, qe = qtail + s.snap[kAppend];
      qtail = qe;
      // T, H: expand the owned frontier into the claims bitmap
      int tile_sz = kBlock;
      while (tile_sz > 32 && (long long)(qe - qs) < (long long)tile_sz * cta_count(Q)) tile_sz >>= 1;
      int64_t chunk = kChunkMax;
      while (chunk > kChunkMin && scout < chunk * nwarps) chunk >>= 1;
      long long sacc = 0, cacc = 0;
      const bool own = Q.own_list != nullptr;
      td_light<true>(Q, s, ph, qapp(Q, ph, qtail), qs, qe, claims, lvl, encode, sacc, qcnt, tile_sz, chunk, false, true,
                     0, 0xffffffffu, own);
      if (!xsync(Q, T, s, ph, xph, kTagTD)) return;
      if (s.snap[kWork]) {  // some rank registered hubs or heavy chunks
        const unsigned long long nch = s.snap[kChunkCount], nown = own ? s.snap[kOwnCount] : 0;
        // hubs: this rank's CTAs each take a range of all n target ids (the
        // claims bitmap's slice in shared memory), parents stored window by
        // window into the owners' arrays
        if (nown) td_own(Q, s, nown, claims, wsm);
        td_heavy<true>(Q, s, ph, qapp(Q, ph, qtail), nch, claims, lvl, encode, sacc, qcnt, false);
        if (!xsync(Q, T, s, ph, xph, kTagHeavy)) return;
      }
      // S: owners merge every rank's claims over their words
      sacc = 0;
      merge_claims(Q, T, r, nextg, lvl, sacc, cacc);
      const unsigned set = ph & 3;
      block_add(sacc, &Q.ctrl->cnt[set][kSum], s);
      block_add(cacc, &Q.ctrl->cnt[set][kCount], s);
      if (!xsync(Q, T, s, ph, xph, kTagSweep)) return;
      scout = (long long)s.snap[kSum];
      const long long claimed = (long long)s.snap[kCount];
      if (T.nranks > 1) {
        broadcast_owned(Q, T, r, 2 - cur, gtid, gthreads);  // all-gather of next
        if (!xsync(Q, T, s, ph, xph, kTagZero)) return;
      }
      reached += claimed;
      gfront = claimed;
      // kTopDownRescan (bfs.hpp:161-167) totals the new frontier's degrees:
      // on an undirected graph every claimed vertex has degree >= 1, so
      // that total equals the encoded sum above
      log_step(Q, nsteps++, 'T', fsize, scout, etc);
      lvl++;
      cur ^= 1;
    }
  }
  if (cta_id(Q) == 0 && threadIdx.x == 0) {
    Q.ctrl->num_steps = nsteps;
    Q.ctrl->xsyncs = xph;
  }
}

}  // namespace

cudaError_t shard_configure(int device, BfsLaunch* cfg) {
  cudaError_t e;
  int sms = 0, coop = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) return e;
  if ((e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device))) return e;
  if (!coop) return cudaErrorNotSupported;
  int optin = 0;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device))) return e;
  const size_t budget = (size_t)optin > sizeof(SmemT) + sizeof(BfsParams) + 1024
                            ? optin - sizeof(SmemT) - sizeof(BfsParams) - 1024 : 0;
  if ((e = cudaFuncSetAttribute(bfs_sharded, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(budget & ~size_t(15)))))
    return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_sharded, kBlock, kBuListBytes))) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  cfg->grid = sms * occ;
  cfg->block = kBlock;
  cfg->smem_static = sizeof(SmemT);
  size_t keep = 0;  // the largest dynamic smem (owned-range slice) that keeps this occupancy
  if ((e = cudaOccupancyAvailableDynamicSMemPerBlock(&keep, bfs_sharded, occ, kBlock))) return e;
  cfg->smem_keep_occ = keep & ~size_t(15);
  return cudaSuccess;
}

cudaError_t shard_launch(const BfsParams& p, const ShardTab& t, int grid, cudaStream_t st) {
  if (cudaError_t e = cudaMemsetAsync(p.ctrl, 0, kCtrlClear, st)) return e;
  BfsParams lp = p;
  ShardTab lt = t;
  void* args[] = {&lp, &lt};
  const size_t dyn = p.own_list ? std::max(kBuListBytes, (size_t)p.own_span_w * 4) : kBuListBytes;
  return cudaLaunchCooperativeKernel((const void*)bfs_sharded, dim3(grid), dim3(kBlock), args, dyn, st);
}

}  // namespace gk
