// gk_bfs_grid.cuh -- the persistent grid kernel's body (bfs_persistent),
// instantiated in two translation units: gk_bfs_kernel.cu (a fresh
// traversal) and gk_bfs_resume.cu (continuing after the cluster kernel).
// One instantiation per TU keeps the inlining decisions of the fresh
// kernel's code unchanged (two in one TU cost 30% more spill traffic).
#ifndef GK_BFS_GRID_CUH_
#define GK_BFS_GRID_CUH_
#include "gk_bfs_steps.cuh"

namespace gk {
namespace {

#ifndef GK_SPARSE
#define GK_SPARSE 1
#endif
#ifndef GK_INIT_MODE_DEF
#define GK_INIT_MODE_DEF 1
#endif
#ifndef GK_PUSH_BU
#define GK_PUSH_BU 1
#endif
#ifndef GK_PUSH_FACTOR
#define GK_PUSH_FACTOR 8
#endif
#ifndef GK_CM_HANDOFF
#define GK_CM_HANDOFF 1
#endif
constexpr int kCmEnter = 8;  // tiny top-down steps in a row before the cluster kernel takes over
constexpr long long kPushFactor = GK_PUSH_FACTOR;  // pushed bottom-up step when scout < this x pending
// kResume: the launch continues a traversal the cluster kernel handed back
// (a separate instantiation, so the fresh traversal's code is unchanged).
template <bool kResume>
#ifndef GK_MINB
#define GK_MINB 2  // CTAs per SM the register allocation must allow (64 registers at 2)
#endif
__global__ void __launch_bounds__(kBlock, GK_MINB) bfs_persistent(BfsParams P) {
  extern __shared__ uint4 dyn_smem[];
  __shared__ SmemT s;
  unsigned ph = 0;
  const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gthreads = (long long)gridDim.x * kBlock;
  const uint32_t src = P.src;

  // ---- init (timed; replaces bfs.hpp:126-138) ----
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->ts[0] = globaltimer();
  if (!kResume) {  // a resumed traversal keeps its state
    const long long n4 = P.n >> 2;
    int4* p4 = reinterpret_cast<int4*>(P.parent);
    int4* d4 = reinterpret_cast<int4*>(P.depth);
    const int4 m1 = make_int4(-1, -1, -1, -1);
    if (!P.parent_preset) {
#pragma unroll 4
      for (long long i = gtid; i < n4; i += gthreads) p4[i] = m1;
      for (long long i = (n4 << 2) + gtid; i < P.n; i += gthreads) P.parent[i] = -1;
    }
    if (P.want_depth) {
      for (long long i = gtid; i < n4; i += gthreads) d4[i] = m1;
      for (long long i = (n4 << 2) + gtid; i < P.n; i += gthreads) P.depth[i] = -1;
    }
    // visited starts as the never-reachable set, so sweeps skip it
    const long long w4 = P.w32 >> 2;
    for (long long i = gtid; i < w4; i += gthreads) {
      reinterpret_cast<uint4*>(P.visited)[i] = __ldg(reinterpret_cast<const uint4*>(P.dead) + i);
    }
    for (long long i = (w4 << 2) + gtid; i < P.w32; i += gthreads) {
      P.visited[i] = __ldg(P.dead + i);
    }
  }
  if (!kResume) {
    if (!grid_sync(P, s, ph, kTagInit)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // bfs.hpp:132-136
      P.parent[src] = (int32_t)src;
      if (P.want_depth) P.depth[src] = 0;
      P.visited[src >> 5] |= 1u << (src & 31u);
      P.queue[0] = src;
    }
    if (!grid_sync(P, s, ph, kTagInit)) return;
  }

  const bool encode = P.strategy != GK_BFS_TOP_DOWN_RESCAN;
  unsigned long long qs = 0, qe = 1;
  unsigned long long qtail = 1;  // queue entries written so far (uniform)
  long long etc = P.m;                                  // bfs.hpp:139
  long long scout = offv(P, P.out_off, src + 1) - offv(P, P.out_off, src);  // bfs.hpp:140
  long long nsteps = 0;
  long long reached = 1;  // vertices claimed so far (source included)
  long long dummy = 0;
  int ntiny = 0;  // consecutive tiny top-down steps (cluster-mode hand-off)
  // sparse sweeps while few vertices are pending (and the list scratch holds them twice)
#ifndef GK_SPARSE_MUL
#define GK_SPARSE_MUL 1  // sparse sweeps while pending <= GK_SPARSE_MUL * n/32
#endif
  auto sparse_ok = [&](long long pend) {
    return !P.front_in_smem && GK_SPARSE && pend <= GK_SPARSE_MUL * P.w32 && 2 * pend <= 4 * P.chunk_cap;
  };
  int lvl = 0;
  int qcnt = 0;
  bool front_ready = false;  // frontg holds exactly the current frontier
  bool queue_stale = false;  // the current frontier's queue window is not written yet
  uint32_t* frontg = P.bm0;
  uint32_t* nextg = P.bm1;
  if (kResume) {  // continue where the cluster kernel handed back (P.rs)
    qs = (unsigned long long)P.rs.qs;
    qe = (unsigned long long)P.rs.qe;
    qtail = (unsigned long long)P.rs.qtail;
    etc = P.rs.etc;
    scout = P.rs.scout;
    nsteps = P.rs.nsteps;
    reached = P.rs.reached;
    lvl = (int)P.rs.lvl;
    if (P.rs.swap) {
      frontg = P.bm1;
      nextg = P.bm0;
    }
  }
  uint32_t* sfront = reinterpret_cast<uint32_t*>(dyn_smem);
  const long long nwarps = gthreads >> 5;
  int bu_tw_log = P.bu_tw_log_max;  // bottom-up task = 32 words unless that leaves warps idle
  while (bu_tw_log > 0 && ((P.w32 + (1 << bu_tw_log) - 1) >> bu_tw_log) < nwarps) bu_tw_log--;

  // A large top-down step over the queue window [a, b) whose frontier's
  // out-degree total is sc: next := visited, bitmap claims (owned-range hub
  // expansion, light tiles, heavy chunks; target-range passes when next
  // exceeds L2), then the claim sweep.  Leaves the claims in nextg (visited
  // updated); claimed / sc_out are grid totals.
  auto large_step = [&](unsigned long long a, unsigned long long b, long long sc, unsigned long long& claimed,
                        long long& sc_out) -> bool {
    for (long long i = gtid; i < P.w32; i += gthreads) nextg[i] = __ldcg(P.visited + i);
    if (!grid_sync(P, s, ph, kTagZero)) return false;
    int tile_sz = kBlock;
    while (tile_sz > 32 && (long long)(b - a) < (long long)tile_sz * gridDim.x) tile_sz >>= 1;
    int64_t chunk = kChunkMax;
    while (chunk > kChunkMin && sc < chunk * nwarps) chunk >>= 1;
    long long sacc = 0;
    // Claims only touch next (n/8 bytes).  When that bitmap is larger than
    // L2 can hold, the step runs in P.td_passes passes over target vertex
    // ranges of P.td_span ids, each pass's slice of next (and of parent)
    // staying L2-resident; the frontier's lists are re-streamed per pass,
    // which HBM does at full bandwidth.
    unsigned long long nch = 0, nown = 0;
    const bool own = P.own_list != nullptr && P.td_passes == 1;
    for (int r = 0; r < P.td_passes; r++) {
      const uint32_t rlo = (uint32_t)((int64_t)r * P.td_span);
      const uint32_t rhi = r + 1 == P.td_passes ? 0xffffffffu : (uint32_t)((int64_t)(r + 1) * P.td_span);
      {
        const QApp qa = qapp(P, ph, qtail);
        td_light<true>(P, s, ph, qa, a, b, nextg, lvl, encode, sacc, qcnt, tile_sz, chunk, false, r == 0, rlo,
                       rhi, own);
      }
      if (!grid_sync(P, s, ph, kTagTD)) return false;
      if (r == 0) {
        nch = s.snap[kChunkCount];
        nown = own ? s.snap[kOwnCount] : 0;
      }
      if (nch || nown) {
        if (nown) td_own(P, s, nown, nextg, sfront);
        const QApp qa = qapp(P, ph, qtail);
        if (nch) td_heavy<true>(P, s, ph, qa, nch, nextg, lvl, encode, sacc, qcnt, false, rlo, rhi);
        if (!grid_sync(P, s, ph, nown ? kTagOwn : kTagHeavy)) return false;
      }
    }
    long long cacc = 0;
    sacc = 0;
    const unsigned set = ph & 3;
    td_scout_bits(P, nextg, lvl, encode, sacc, cacc);
    block_add(sacc, &P.ctrl->cnt[set][kSum], s);
    block_add(cacc, &P.ctrl->cnt[set][kCount], s);
    if (!grid_sync(P, s, ph, kTagSweep)) return false;
    sc_out = (long long)s.snap[kSum];
    claimed = s.snap[kCount];
    return true;
  };

  while (qe > qs) {
    const bool go_bu = P.strategy == GK_BFS_DIRECTION_OPTIMIZING && scout > etc / P.alpha;
    // a top-down step whose (bitmap) frontier outnumbers the pending
    // vertices is executed as a sparse pull (see sparse_step)
    const bool pull = !go_bu && P.strategy == GK_BFS_DIRECTION_OPTIMIZING && front_ready &&
                      P.live - reached <= (long long)(qe - qs) && sparse_ok(P.live - reached);
    if (!go_bu && !pull && queue_stale) {  // BitmapToQueue for the coming top-down step
      b2q(P, qapp(P, ph, qtail), frontg);
      if (!grid_sync(P, s, ph, kTagB2Q)) return;
      qtail += s.snap[kAppend];
      queue_stale = false;
    }
    if (go_bu || pull) ntiny = 0;
    // A chain of tiny top-down steps (high-diameter graphs) continues in the
    // cluster kernel (gk_bfs_cluster.cu): hand the state to the host loop.
    if (GK_CM_HANDOFF && P.cm_ok && !go_bu && !pull && ntiny >= kCmEnter && scout <= P.cm_max_scout && scout <= kTinyStep &&
        scout <= P.bitmap_td_min && (long long)(qe - qs) <= kTinyFrontier) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        Hand& h = P.ctrl->hand;
        h.qs = (long long)qs;
        h.qe = (long long)qe;
        h.qtail = (long long)qtail;
        h.etc = etc;
        h.scout = scout;
        h.nsteps = nsteps;
        h.reached = reached;
        h.lvl = lvl;
        h.swap = frontg == P.bm1;
        h.mode = 1;
        P.ctrl->num_steps = nsteps;
      }
      return;
    }
    if (go_bu) {
      // A bottom-up step whose frontier's out-degree total (scout, known after
      // a top-down step) is small against the vertices still pending runs as
      // a large top-down step (push): same claimed set and awake count;
      // parents are any frontier in-neighbour instead of the first in
      // ascending order (bfs.hpp:55-60) -- valid parents either way.  The
      // pull would scan the whole in-list of every pending vertex without a
      // frontier neighbour (kron27: the sources whose first bottom-up step
      // follows two top-down steps from a few hubs, 3.2 -> 2.0 ms).  The 8x
      // bound is measured: a cost model (pull tests ~min(mean degree,
      // m / scout) arcs per pending vertex) pushed urand27 steps where the
      // pull is faster, and pushing from a bitmap-only frontier (after a
      // large top-down step) never paid.
      bool push_first = GK_PUSH_BU && !queue_stale && !P.front_in_smem && !sparse_ok(P.live - reached) &&
                        scout < kPushFactor * (P.live - reached);
      const unsigned long long fq0 = qs, fq1 = qe;
      if (!front_ready && !push_first) {  // QueueToBitmap into a cleared front (bfs.hpp:145)
        for (long long i = gtid; i < P.w32; i += gthreads) frontg[i] = 0u;
        if (!grid_sync(P, s, ph, kTagZero)) return;
        for (unsigned long long i = qs + gtid; i < qe; i += gthreads) {
          const uint32_t v = __ldcg(P.queue + i);
          atomicOr(frontg + (v >> 5), 1u << (v & 31u));
        }
        if (!grid_sync(P, s, ph, kTagQ2B)) return;
      }
      long long awake = (long long)(qe - qs);  // bfs.hpp:146
      if (queue_stale) {  // the bitmap-only frontier's queue window is never written
        qe = qtail;
        queue_stale = false;
      }
      qs = qe;  // bfs.hpp:147
      long long old_awake;
      do {  // bfs.hpp:149-154
        old_awake = awake;
        const uint32_t* fr = frontg;
        if (P.front_in_smem) {
          for (long long i = threadIdx.x; i < P.w32; i += kBlock) sfront[i] = __ldcg(frontg + i);
          __syncthreads();
          fr = sfront;
        }
        long long acc = 0;
        if (push_first) {
          push_first = false;
          unsigned long long claimed = 0;
          long long sdummy = 0;
          if (!large_step(fq0, fq1, scout, claimed, sdummy)) return;
          awake = (long long)claimed;
          reached += awake;
          log_step(P, nsteps++, 'B', old_awake, awake, etc, 'P');
          lvl++;
          uint32_t* t = frontg;
          frontg = nextg;
          nextg = t;
          continue;
        }
        if (sparse_ok(P.live - reached)) {
          long long found = 0;
          if (!sparse_step<false>(P, s, ph, frontg, nextg, lvl, found, dummy)) return;
          awake = found;
          reached += awake;
          log_step(P, nsteps++, 'B', old_awake, awake, etc);
          lvl++;
          uint32_t* t = frontg;
          frontg = nextg;
          nextg = t;
          continue;
        }
        // long-list scratch: queue slots past the tail are unused during bottom-up
        const unsigned long long lbase = qe;
        if (P.front_in_smem) bu_step<true>(P, s, ph, fr, nextg, lvl, lbase, bu_tw_log, acc, nullptr);
        else bu_step<false>(P, s, ph, fr, nextg, lvl, lbase, bu_tw_log, acc, sfront);
        unsigned set = ph & 3;
        block_add(acc, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagBU)) return;
        const unsigned long long nlong = s.snap[kLongCount];
        long long awake_bu = (long long)s.snap[kSum];
        if (nlong) {
          acc = 0;
          if (P.front_in_smem) bu_long<true>(P, fr, nextg, P.queue + lbase, nlong, lvl, acc, dummy);
          else bu_long<false>(P, fr, nextg, P.queue + lbase, nlong, lvl, acc, dummy);
          set = ph & 3;
          block_add(acc, &P.ctrl->cnt[set][kSum], s);
          if (!grid_sync(P, s, ph, kTagLong)) return;
          awake_bu += (long long)s.snap[kSum];
        }
        awake = awake_bu;
        reached += awake;
        log_step(P, nsteps++, 'B', old_awake, awake, etc);
        lvl++;
        uint32_t* t = frontg;
        frontg = nextg;
        nextg = t;
      } while (awake >= old_awake || awake > P.n / P.beta);
      if (P.live - reached <= awake && sparse_ok(P.live - reached)) {
        // the coming top-down step is pulled (see above): no queue needed
        qs = qtail;
        qe = qtail + awake;
        queue_stale = true;
      } else {
        b2q(P, qapp(P, ph, qtail), frontg);  // bfs.hpp:155
        if (!grid_sync(P, s, ph, kTagB2Q)) return;
        qtail += s.snap[kAppend];
        qe = qtail;
      }
      scout = 1;  // bfs.hpp:156
      front_ready = true;
    } else {
      etc -= scout;  // bfs.hpp:158
      const long long fsize = (long long)(qe - qs);
      if (pull) {
        long long claimed = 0, sc = 0;
        if (!sparse_step<true>(P, s, ph, frontg, nextg, lvl, claimed, sc)) return;
        scout = sc;
        reached += claimed;
        uint32_t* t = frontg;
        frontg = nextg;
        nextg = t;
        front_ready = true;
        qs = qtail;  // bitmap-only frontier, as after a large top-down step
        qe = qtail + claimed;
        queue_stale = true;
        log_step(P, nsteps++, 'T', fsize, scout, etc, 'U');
        lvl++;
        continue;
      }
      const unsigned long long qt0 = qtail;
      // Large frontiers (by the degree total the heuristic already holds)
      // also build the next-frontier bitmap and sum degrees in a separate
      // high-MLP pass; small ones keep everything inline, so a long chain of
      // tiny levels costs one grid barrier each.
      const bool big = scout > P.bitmap_td_min;
      // (after a bottom-up phase scout is 1, bfs.hpp:156: the frontier size
      // bounds the step then)
      const bool tiny = scout <= kTinyStep && fsize <= kTinyFrontier;
      // Granularity from the step size the heuristic already knows: enough
      // tiles / chunks for every CTA / warp (hardware-derived, not per graph).
      int tile_sz = kBlock;
      while (tile_sz > 32 && (long long)(qe - qs) < (long long)tile_sz * gridDim.x) tile_sz >>= 1;
      int64_t chunk = kChunkMax;
      while (chunk > kChunkMin && scout < chunk * nwarps) chunk >>= 1;
      long long sacc = 0;
      unsigned set;
      if (big) {
        unsigned long long claimed = 0;
        if (!large_step(qs, qe, scout, claimed, scout)) return;
        reached += (long long)claimed;
        uint32_t* t = frontg;
        frontg = nextg;
        nextg = t;
        front_ready = true;
        // The new frontier exists only as a bitmap; its queue window is
        // [qtail, qtail + claimed), materialised by BitmapToQueue only if a
        // top-down step follows.
        qs = qtail;
        qe = qtail + claimed;
        queue_stale = true;
      } else {
        set = ph & 3;
        {
          const QApp qa = qapp(P, ph, qtail);
          td_light<false>(P, s, ph, qa, qs, qe, nextg, lvl, encode, sacc, qcnt, tile_sz, chunk, tiny);
          wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
        }
        block_add(sacc, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagTD)) return;
        scout = (long long)s.snap[kSum];
        qtail += s.snap[kAppend];
        const unsigned long long nch = s.snap[kChunkCount];
        if (nch) {
          sacc = 0;
          set = ph & 3;
          const QApp qa = qapp(P, ph, qtail);
          td_heavy<false>(P, s, ph, qa, nch, nextg, lvl, encode, sacc, qcnt, tiny);
          wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
          block_add(sacc, &P.ctrl->cnt[set][kSum], s);
          if (!grid_sync(P, s, ph, kTagHeavy)) return;
          scout += (long long)s.snap[kSum];
          qtail += s.snap[kAppend];
        }
      }
      if (!big) {
        front_ready = false;
        reached += (long long)(qtail - qt0);
        qs = qe;  // SlideWindow (bfs.hpp:160)
        qe = qtail;
      }
      if (P.strategy == GK_BFS_TOP_DOWN_RESCAN) {  // bfs.hpp:161-167
        long long tot = 0;
        for (unsigned long long i = qs + gtid; i < qe; i += gthreads) {
          const uint32_t u = __ldcg(P.queue + i);
          tot += offv(P, P.out_off, u + 1) - offv(P, P.out_off, u);
        }
        set = ph & 3;
        block_add(tot, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagRescan)) return;
        scout = (long long)s.snap[kSum];
      }
      log_step(P, nsteps++, 'T', fsize, scout, etc);
      lvl++;
      ntiny = tiny && !big ? ntiny + 1 : 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->num_steps = nsteps;
  // bfs.hpp:171-175's final sweep is unnecessary: unreached slots were
  // written -1 by init and never touched.
}

}  // namespace
}  // namespace gk

#endif  // GK_BFS_GRID_CUH_
