// gk_bfs_cluster.cu -- cluster mode for long chains of tiny top-down levels
// (high-diameter graphs: SURVEY.md §7 hard part 7, config 4).
//
// In the grid kernel (bfs_persistent) a tiny top-down level is a chain of
// dependent accesses -- queue entry, its offsets, its list, the claim, the
// queue append, the counters -- closed by a 296-CTA grid barrier: ~10 us per
// level, thousands of levels on a road graph.  When the direction heuristic
// has chosen kCmEnter tiny top-down steps in a row, the grid kernel hands the
// traversal to this kernel: ONE thread-block cluster (16 or 8 CTAs of 512
// threads) that runs the same levels with
//   * the frontier in distributed shared memory: a claimed vertex travels,
//     with its offset and degree (read together with the claim atomic), to
//     the CTA its id hashes to, so the next level starts from shared memory
//     with balanced CTAs and no offset reload;
//   * no cluster-wide barrier: entries and per-level totals are st.async
//     stores into the destination's shared memory whose completion is
//     counted on the destination's mbarrier (complete_tx), so a CTA starts
//     the next level as soon as ITS inputs have landed (a cluster barrier
//     orders global memory too: MEMBAR.GPU per level).
// Claims, parents, depths and the step log are the grid kernel's (visited
// bitmap in global memory, parent stores, bfs.hpp:77-84 semantics); the
// reference's schedule and counters are kept exactly.  The kernel hands back
// (Hand, gk_internal.cuh) when the traversal ends, when the heuristic turns
// to a bottom-up or a non-tiny step, or when a sender's region for a
// destination overflows (the overflow goes to the global queue, so no claim
// is lost).  The host loop in gk_capi.cu (run_handoffs) launches whichever
// kernel the hand-off names, inside the trial's timed region.
#include <cooperative_groups.h>

#include "gk_persistent.cuh"

namespace gk {
namespace {

namespace cg = cooperative_groups;

constexpr int kCmBlock = 512;  // 128 registers per thread: the level state stays out of local memory
constexpr int kCmCap = 4096;  // frontier entries per CTA per array

struct CmEnt {
  uint32_t v;
  uint32_t deg;
  int64_t off;
};

constexpr uint32_t kCmLight = 16;  // lists up to this long are expanded by their own lane
constexpr int kCmW = 4;            // arcs per lane in flight
constexpr int kCmSub = 4;          // sub-regions per (sender, destination) region

struct CmArc {  // one arc of a flattened short list: parent, position in the neighbour array
  uint32_t u;
  uint32_t pad;
  int64_t pos;
};

// Messages between the CTAs of the cluster (DSMEM, no cluster barrier per
// level).  During level L every CTA sends each CTA d (itself included):
//   * the claimed vertices whose home is d, as 16-byte entries stored with
//     st.async into d's region for this sender, f[(L+1)&1][sender];
//   * one header {entries sent, claims, scout low 16 bits, scout >> 16 |
//     overflow << 31} into d's hdr[(L+1)&1][sender];
//   * one arrival on d's mbar[(L+1)&1] announcing those bytes (expect_tx).
// d's barrier phase completes once all C senders arrived and all their bytes
// landed, so d starts level L+1 when ITS inputs are complete -- the CTAs
// drift apart by at most one level, which the parity double buffers absorb
// (a sender of level L+1 messages has received d's level-L header, sent
// after d finished reading the buffers it overwrites).
struct __align__(16) CmShared {
  CmEnt f[2][kCmCap];          // [parity][sender region of kCmCap / C entries]
  uint4 hdr[2][16];            // [parity][sender]
  unsigned long long mbar[2];  // per parity, C arrivals per phase
  unsigned long long ctot[2][2];  // this CTA's level totals by send parity: claims, scout
  unsigned lc[2][16][kCmSub];  // entries sent per destination and sub-region, by send parity
  unsigned lovf[2];            // an entry of this CTA went to the global queue
  // kTopDownRescan's extra pass (bfs.hpp:161-167): per-CTA degree totals of
  // the new frontier, exchanged like the headers on their own barriers
  uint4 rmsg[2][16];
  unsigned long long rbar[2];
  unsigned long long rsum[2];
  CmArc arc[kCmBlock / 32][32 * kCmW];  // per warp: the short lists being claimed
  unsigned dbg[2][4];  // GK_CM_TRACE == 2: per-level warp timing of CTA 0
  unsigned dbs[2][4];  // sub-phases of a warp's first round
};


#ifndef GK_CM_TRACE
#define GK_CM_TRACE 0  // diagnostics: 1 CTA 0 logs per-level phase cycles in the trace, 2 its warp timing
#endif
#if GK_CM_TRACE == 1
// the clock is read once dep (a register) is available
#define CM_MARKD(i, dep)                                                                    \
  do {                                                                                      \
    if (c == 0 && t == 0 && L < 120) {                                                      \
      unsigned long long ck_;                                                               \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck_) : "r"((unsigned)(dep)));            \
      P.ctrl->ts[L * 4 + (i)] = ck_;                                                        \
      P.ctrl->tag[L * 4 + (i)] = 'a' + (i);                                                 \
    }                                                                                       \
  } while (0)
#else
#define CM_MARKD(i, dep) \
  do {                   \
  } while (0)
#endif
#define CM_MARK(i) CM_MARKD(i, 0u)

__device__ __forceinline__ unsigned cm_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cm_mapa(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// 16 bytes into another CTA's shared memory, completion counted on its barrier
__device__ __forceinline__ void cm_st_async(unsigned ra, uint32_t x, uint32_t y, uint32_t z, uint32_t w,
                                            unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
               "r"(x), "r"(y), "r"(z), "r"(w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cm_arrive_tx(unsigned rbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool cm_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n }"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Home CTA of a vertex: a mixing hash (a multiplicative one maps the fixed
// id offsets of a mesh's neighbours to fixed CTA offsets, so a sender's
// claims piled up in a few of its regions).
__device__ __forceinline__ int cm_home(uint32_t v, int lgc) {
  v ^= v >> 16;
  v *= 0x85ebca6bu;
  v ^= v >> 13;
  v *= 0xc2b2ae35u;
  v ^= v >> 16;
  return lgc ? (int)(v >> (32 - lgc)) : 0;
}

// scout > etc / alpha (bfs.hpp:143) without a 64-bit division when the
// product cannot overflow: for etc >= 0 and integer scout the two agree.
__device__ __forceinline__ bool cm_go_bu(const BfsParams& P, long long scout, long long etc) {
  if (P.strategy != GK_BFS_DIRECTION_OPTIMIZING) return false;
  if (etc >= 0 && P.alpha < (1 << 20) && scout < (1ll << 40)) return scout * P.alpha > etc;
  return scout > etc / P.alpha;
}

__global__ void __launch_bounds__(kCmBlock, 1) bfs_cluster(BfsParams P, Hand H) {
  extern __shared__ uint4 cm_dsm[];
  CmShared& S = *reinterpret_cast<CmShared*>(cm_dsm);
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), C = (int)cl.num_blocks();
  int lgc = 0;
  while ((1 << lgc) < C) lgc++;
  const int R = kCmCap / C;  // entries per sender region
  const int t = threadIdx.x;
  const unsigned lane = t & 31u, warp = t >> 5;
  const long long base = H.qtail;  // hand-back window starts here
  const unsigned f_sa = cm_saddr(&S.f[0][0]), hdr_sa = cm_saddr(&S.hdr[0][0]), bar_sa = cm_saddr(&S.mbar[0]);
  if (t < 4) (&S.ctot[0][0])[t] = 0ull;
  if (t < 2 * 16 * kCmSub) (&S.lc[0][0][0])[t] = 0u;
  const unsigned rmsg_sa = cm_saddr(&S.rmsg[0][0]), rbar_sa = cm_saddr(&S.rbar[0]);
  if (t < 2) {
    S.lovf[t] = 0u;
    S.rsum[t] = 0ull;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_sa + 8u * t), "r"(C) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rbar_sa + 8u * t), "r"(C) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cl.sync();
  const bool encode = P.strategy != GK_BFS_TOP_DOWN_RESCAN;
  long long etc = H.etc, scout = H.scout, nsteps = H.nsteps, reached = H.reached, fr = H.qe - H.qs;
  int lvl = (int)H.lvl;
  unsigned L = 0;
  unsigned long long t0 = 0;
  if (t == 0) t0 = globaltimer();

  // a claimed (or loaded) vertex to its home CTA's region for this sender:
  // slot idx of sub-region sub (warps w with w % kCmSub == sub share one, so
  // fewer warps contend for each local counter)
  const int R4 = R / kCmSub;
  const int sub = (int)warp & (kCmSub - 1);
  auto push_at = [&](int dp, int home, unsigned idx, uint32_t v, uint32_t deg, int64_t off) {
    if (idx < (unsigned)R4) {
      const unsigned slot = (unsigned)(dp * kCmCap + c * R + sub * R4 + (int)idx);
      cm_st_async(cm_mapa(f_sa + slot * (unsigned)sizeof(CmEnt), home), v, deg, (uint32_t)off,
                  (uint32_t)((uint64_t)off >> 32), cm_mapa(bar_sa + 8u * dp, home));
    } else {  // region full: to the global queue; the traversal returns to the grid kernel
      P.queue[base + atomicAdd(&P.ctrl->hand.qfill, 1ull)] = v;
      S.lovf[dp] = 1u;
    }
  };
  auto push = [&](int dp, uint32_t v, uint32_t deg, int64_t off) {
    const int home = cm_home(v, lgc);
    push_at(dp, home, atomicAdd(&S.lc[dp][home][sub], 1u), v, deg, off);
  };
  // after every warp's pushes and totals of send parity dp: headers + arrivals to every CTA
  auto send = [&](int dp) {
    __syncthreads();
    if (warp == 0) {
      const unsigned long long cc = S.ctot[dp][0], sc = S.ctot[dp][1];
      const unsigned of = S.lovf[dp];
      if ((int)lane < C) {
        unsigned packed = 0, sent = 0;
#pragma unroll
        for (int k = 0; k < kCmSub; k++) {
          const unsigned n = S.lc[dp][lane][k];
          packed |= min(n, 255u) << (8 * k);
          sent += min(n, (unsigned)R4);
          S.lc[dp][lane][k] = 0u;
        }
        const unsigned rbar = cm_mapa(bar_sa + 8u * dp, (int)lane);
        cm_st_async(cm_mapa(hdr_sa + (unsigned)(dp * 16 + c) * 16u, (int)lane), packed, (uint32_t)cc,
                    (uint32_t)(sc & 0xffff), (uint32_t)(sc >> 16) | (of << 31), rbar);
        cm_arrive_tx(rbar, 16u * (1u + sent));
      }
      __syncwarp();
      if (lane == 0) {
        S.ctot[dp][0] = S.ctot[dp][1] = 0ull;
        S.lovf[dp] = 0u;
      }
    }
  };

  // the frontier's queue window into the home CTAs' level-0 regions
  {
    unsigned loaded = 0;
    for (long long i = H.qs + (long long)c * kCmBlock + t; i < H.qe; i += (long long)C * kCmBlock) {
      const uint32_t v = __ldcg(P.queue + i);
      const int64_t o0 = offv(P, P.out_off, v), o1 = offv(P, P.out_off, v + 1);
      push(0, v, (uint32_t)(o1 - o0), o0);
      loaded++;
    }
    const unsigned wl = __reduce_add_sync(kFull, loaded);
    if (lane == 0 && wl) atomicAdd(&S.ctot[0][0], (unsigned long long)wl);
    send(0);
  }

  // warp w walks sender region w % C, every wpr-th group of 32 entries
  const int reg = (int)warp % C, wpr = (kCmBlock / 32) / C, g0 = ((int)warp / C) * 32;
  long long fsize = 0;
  int nr = 0, p1 = 0, p2 = 0, p3 = 0;  // entries of this warp's region at the current level, sub-region prefixes
  // entry e of this warp's region -> its slot in f[parity]
  auto eslot = [&](int e) {
    const int k = (e >= p1) + (e >= p2) + (e >= p3);
    const int b = k == 0 ? 0 : k == 1 ? p1 : k == 2 ? p2 : p3;
    return reg * R + k * R4 + (e - b);
  };
#ifdef GK_CM_EXITTAG
  unsigned dbg_maxn = 0, dbg_bit = 0;
#endif  // entries of this warp's region at the current level
  for (;; L++) {
    const int cur = (int)(L & 1u), nxt = cur ^ 1;
    // wait for this level's frontier (sent during the previous level)
    {
      const unsigned bar = bar_sa + 8u * cur, par = (L >> 1) & 1u;
      unsigned spins = 0;
      while (!cm_try_wait(bar, par)) {
        if (t == 0 && (++spins & 1023u) == 0 && globaltimer() - t0 > P.timeout_ns) {
          atomicExch(&P.ctrl->error, 2);  // watchdog: a sender never arrived
          asm volatile("trap;");
        }
      }
    }
    CM_MARK(0);
#if GK_CM_TRACE == 2
    unsigned xs = 0;
    if (c == 0 && t == 0) {
      const unsigned now = (unsigned)clock64();
      if (L == 0) P.ctrl->ts[0] = 0;
      if (L > 0 && L <= 120) {
        const unsigned* d = S.dbg[(L - 1) & 1];
        P.ctrl->ts[(L - 1) * 4 + 0] = (L == 1 ? 0 : d[0]);
        P.ctrl->ts[(L - 1) * 4 + 1] = d[1] / (kCmBlock / 32);
        const unsigned* d2 = S.dbs[(L - 1) & 1];
        P.ctrl->ts[(L - 1) * 4 + 1] = d2[0];
        P.ctrl->ts[(L - 1) * 4 + 2] = d2[1];
        P.ctrl->ts[(L - 1) * 4 + 3] = d2[2];
        for (int i = 0; i < 4; i++) P.ctrl->tag[(L - 1) * 4 + i] = 'a' + i;
      }
      unsigned* e = S.dbg[(L + 1) & 1];
      e[0] = e[1] = e[2] = 0;
      unsigned* e2 = S.dbs[(L + 1) & 1];
      e2[0] = e2[1] = e2[2] = 0;
    }
    xs = (unsigned)clock64();
    if (c == 0 && t == 0) S.dbg[L & 1][3] = xs;
#endif
    // headers: lane j holds sender j's; totals by warp reductions (same in every warp)
    bool ovf;
    long long claims, sc_next;
    {
      const uint4 h = (int)lane < C ? S.hdr[cur][lane] : make_uint4(0u, 0u, 0u, 0u);
      claims = (long long)__reduce_add_sync(kFull, h.y);
      const unsigned lo = __reduce_add_sync(kFull, h.z), hi = __reduce_add_sync(kFull, h.w & 0x7fffffffu);
      sc_next = ((long long)hi << 16) + (long long)lo;
      bool full = false;  // a sub-region overflowed
#pragma unroll
      for (int k = 0; k < kCmSub; k++) full |= ((h.x >> (8 * k)) & 0xffu) > (unsigned)R4;
      ovf = __any_sync(kFull, (h.w >> 31) != 0u || full);
#ifdef GK_CM_EXITTAG
      dbg_maxn = __reduce_max_sync(kFull, h.x & 0xffu);
      dbg_bit = __reduce_or_sync(kFull, h.w >> 31);
#endif
      const unsigned pk = __shfl_sync(kFull, h.x, reg);
      const int n0 = (int)min(pk & 0xffu, (unsigned)R4), n1 = (int)min((pk >> 8) & 0xffu, (unsigned)R4),
                n2 = (int)min((pk >> 16) & 0xffu, (unsigned)R4), n3 = (int)min(pk >> 24, (unsigned)R4);
      p1 = n0;
      p2 = n0 + n1;
      p3 = p2 + n2;
      nr = p3 + n3;
    }
    if (!encode && L > 0) {
      // kTopDownRescan (bfs.hpp:161-167): the new frontier's degree total by
      // a second pass over it, not from the claims
      const unsigned q = L - 1u, rp = q & 1u;
      unsigned long long mine = 0;
      for (int i = g0 + (int)lane; i < nr; i += wpr * 32) {
        const uint32_t v = S.f[cur][eslot(i)].v;
        mine += (unsigned long long)(offv(P, P.out_off, v + 1) - offv(P, P.out_off, v));
      }
      const unsigned lo = __reduce_add_sync(kFull, (unsigned)(mine & 0xffff));
      const unsigned hi = __reduce_add_sync(kFull, (unsigned)(mine >> 16));
      if (lane == 0 && (lo | hi)) atomicAdd(&S.rsum[rp], ((unsigned long long)hi << 16) + lo);
      __syncthreads();
      if (warp == 0) {
        const unsigned long long tot = S.rsum[rp];
        if ((int)lane < C) {
          const unsigned rb = cm_mapa(rbar_sa + 8u * rp, (int)lane);
          cm_st_async(cm_mapa(rmsg_sa + (rp * 16u + (unsigned)c) * 16u, (int)lane), (uint32_t)(tot & 0xffff),
                      (uint32_t)(tot >> 16), 0u, 0u, rb);
          cm_arrive_tx(rb, 16u);
        }
        __syncwarp();
        if (lane == 0) S.rsum[rp] = 0ull;
      }
      unsigned spins = 0;
      while (!cm_try_wait(rbar_sa + 8u * rp, (q >> 1) & 1u)) {
        if (t == 0 && (++spins & 1023u) == 0 && globaltimer() - t0 > P.timeout_ns) {
          atomicExch(&P.ctrl->error, 2);
          asm volatile("trap;");
        }
      }
      const uint4 m = (int)lane < C ? S.rmsg[rp][lane] : make_uint4(0u, 0u, 0u, 0u);
      sc_next = ((long long)__reduce_add_sync(kFull, m.y) << 16) + (long long)__reduce_add_sync(kFull, m.x);
    }
    if (L > 0) {  // the step log of bfs.hpp:158-160's top-down step L-1
      if (c == 0 && t == 0 && nsteps < P.step_cap) {
        gk_step st;
        st.dir = 'T';
        st.pad = 'K';  // executed by the cluster kernel
        st.frontier = fsize;
        st.result = sc_next;
        st.edges_to_check = etc;
        P.steps[nsteps] = st;
      }
      nsteps++;
      lvl++;
      reached += claims;
      fr = claims;
      scout = sc_next;
    }
    // the same decision as bfs_persistent (bfs.hpp:143-144), uniform in the cluster
    if (fr == 0 || ovf || cm_go_bu(P, scout, etc) || scout > kTinyStep || fr > kTinyFrontier ||
        scout > P.cm_max_scout || scout > P.bitmap_td_min) {
#ifdef GK_CM_EXITTAG  // diagnostic: the last step's tag names why the cluster kernel left
      if (c == 0 && t == 0 && nsteps > 0 && nsteps <= P.step_cap)
        P.steps[nsteps - 1].pad = fr == 0 ? '0' : ovf ? 'o' : cm_go_bu(P, scout, etc) ? 'b' : 'x';
      if (c == 0 && t == 0 && nsteps > 0 && nsteps <= P.step_cap && ovf) {
        P.steps[nsteps - 1].result = dbg_maxn;
        P.steps[nsteps - 1].edges_to_check = dbg_bit * 1000 + L;
      }
#endif
      break;
    }
    etc -= scout;  // bfs.hpp:158
    fsize = fr;
    CM_MARKD(1, nr);
    long long sc = 0;
    unsigned cc = 0;
    // Claims of up to kCmW arcs u -> w per thread, their loads and atomics
    // issued together (bfs.hpp:77-84); the claimed vertex's degree is read
    // with the claim and travels with its frontier entry.
    auto claimw = [&](const uint32_t (&u)[kCmW], const uint32_t (&w)[kCmW], const bool (&ok)[kCmW]) {
#if GK_CM_TRACE == 2
      unsigned t_a = 0;
      asm volatile("mov.u32 %0, %%clock;" : "=r"(t_a) : "r"(w[0] + w[1] + w[kCmW - 1]));
#endif
      int64_t o0[kCmW], o1[kCmW];
#pragma unroll
      for (int q = 0; q < kCmW; q++) {
        o0[q] = o1[q] = 0;
        if (ok[q]) {
          o0[q] = offv(P, P.out_off, w[q]);
          o1[q] = offv(P, P.out_off, w[q] + 1);
        }
      }
      // every claim atomic in flight at once: each result has its own
      // register and is looked at only after the last one was issued
      uint32_t old[kCmW];
#pragma unroll
      for (int q = 0; q < kCmW; q++) {
        old[q] = ~0u;  // predicated atomic: its result stays in its own register
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p atom.global.or.b32 %0, [%1], %3;\n }"
            : "+r"(old[q])
            : "l"(P.visited + (w[q] >> 5)), "r"((unsigned)ok[q]), "r"(1u << (w[q] & 31u))
            : "memory");
      }
#if GK_CM_TRACE == 2
      unsigned t_b = 0, t_c = 0;
      asm volatile("mov.u32 %0, %%clock;" : "=r"(t_b) : "r"(old[0] + old[kCmW - 1] + (unsigned)(o1[0] + o1[kCmW - 1])));
#endif
      bool cl[kCmW];
      int home[kCmW];
      unsigned idx[kCmW];
#pragma unroll
      for (int q = 0; q < kCmW; q++) {
        cl[q] = !((old[q] >> (w[q] & 31u)) & 1u);
        home[q] = 0;
        idx[q] = 0;
        if (!cl[q]) continue;
        P.parent[w[q]] = (int32_t)u[q];
        if (P.want_depth) P.depth[w[q]] = lvl + 1;
        const int64_t dg = o1[q] - o0[q];
        // bfs.hpp:83's -old of the degree-encoded slot (kTopDownRescan
        // counts the new frontier's degrees in a separate pass)
        sc += encode ? (dg ? dg : 1) : 0;
        cc++;
        if (dg) {
#if GK_CM_TOUCH  // A/B: a discarded load instead of the L2 prefetch
          uint32_t dummy;
          asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(dummy) : "l"(P.out_nb + o0[q]));
#else
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.out_nb + o0[q]));
#endif
        }
        home[q] = cm_home(w[q], lgc);
        idx[q] = atomicAdd(&S.lc[nxt][home[q]][sub], 1u);
      }
#pragma unroll
      for (int q = 0; q < kCmW; q++)
        if (cl[q]) push_at(nxt, home[q], idx[q], w[q], (uint32_t)(o1[q] - o0[q]), o0[q]);
#if GK_CM_TRACE == 2
      asm volatile("mov.u32 %0, %%clock;" : "=r"(t_c) : "r"((unsigned)cc));
      if (c == 0) {
        const unsigned m = __activemask();
        const unsigned da = __reduce_max_sync(m, t_a - xs), db = __reduce_max_sync(m, t_b - t_a),
                       dc = __reduce_max_sync(m, t_c - t_b);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(m) - 1)) {
          atomicMax(&S.dbs[L & 1][0], da);
          atomicMax(&S.dbs[L & 1][1], db);
          atomicMax(&S.dbs[L & 1][2], dc);
        }
      }
#endif
    };
    // Expansion: warp w walks region w % C (every wpr-th group of 32
    // entries).  The short lists of a group are flattened into the warp's
    // arc buffer (each lane scatters its own, at its prefix) and claimed
    // kCmW arcs per lane at a time, so every lane carries the same load; the
    // long lists are walked by the whole warp together.
    CmArc* ab = S.arc[warp];
    for (int e0 = g0; e0 < nr; e0 += wpr * 32) {
      const int ei = e0 + (int)lane;
      CmEnt en{0u, 0u, 0};
      if (ei < nr) en = S.f[cur][eslot(ei)];
      const bool heavy = en.deg > kCmLight;
      const int dl = heavy ? 0 : (int)en.deg;
      int incl = dl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if ((int)lane >= o) incl += y;
      }
      const int excl = incl - dl, tot = __shfl_sync(kFull, incl, 31);
      for (int b = 0; b < tot; b += 32 * kCmW) {
        const int lo = max(0, b - excl), hi = min(dl, b + 32 * kCmW - excl);
        for (int d = lo; d < hi; d++) ab[excl + d - b] = CmArc{en.v, 0u, en.off + d};
        __syncwarp();
        uint32_t u[kCmW], w[kCmW];
        bool ok[kCmW];
#pragma unroll
        for (int q = 0; q < kCmW; q++) {
          const int j = q * 32 + (int)lane;
          ok[q] = b + j < tot;
          u[q] = w[q] = 0u;
          if (ok[q]) {
            const CmArc a = ab[j];
            u[q] = a.u;
            w[q] = ld_nb(P.out_nb + a.pos);
          }
        }
        __syncwarp();
        claimw(u, w, ok);
      }
      for (unsigned hm = __ballot_sync(kFull, heavy); hm; hm &= hm - 1) {
        const int h = __ffs(hm) - 1;
        const uint32_t hv = __shfl_sync(kFull, en.v, h), hd = __shfl_sync(kFull, en.deg, h);
        const int64_t ho = __shfl_sync(kFull, en.off, h);
        for (uint32_t d0 = 0; d0 < hd; d0 += 32 * kCmW) {
          uint32_t u[kCmW], w[kCmW];
          bool ok[kCmW];
#pragma unroll
          for (int q = 0; q < kCmW; q++) {
            const uint32_t j = d0 + q * 32 + lane;
            ok[q] = j < hd;
            u[q] = hv;
            w[q] = ok[q] ? ld_nb(P.out_nb + ho + j) : 0u;
          }
          claimw(u, w, ok);
        }
      }
    }
    CM_MARKD(2, (unsigned)sc);
#if GK_CM_TRACE == 2
    if (c == 0 && lane == 0) {
      unsigned now;
      asm volatile("mov.u32 %0, %%clock;" : "=r"(now) : "r"((unsigned)sc));
      atomicMax(&S.dbg[L & 1][0], now - xs);
      atomicAdd(&S.dbg[L & 1][1], now - xs);
      atomicMax(&S.dbg[L & 1][2], now);
    }
#endif
    {  // this CTA's totals: warp reductions, shared atomics
      const unsigned wc = __reduce_add_sync(kFull, cc);
      const unsigned lo = __reduce_add_sync(kFull, (unsigned)(sc & 0xffff));
      const unsigned hi = __reduce_add_sync(kFull, (unsigned)(sc >> 16));
      if (lane == 0) {
        if (wc) atomicAdd(&S.ctot[nxt][0], (unsigned long long)wc);
        const unsigned long long ws = ((unsigned long long)hi << 16) + lo;
        if (ws) atomicAdd(&S.ctot[nxt][1], ws);
      }
    }
    send(nxt);
    CM_MARK(3);
  }
  // hand back: the current entries join the global queue after the overflow
  {
    for (int i = g0 + (int)lane; i < nr; i += wpr * 32)
      P.queue[base + atomicAdd(&P.ctrl->hand.qfill, 1ull)] = S.f[L & 1u][eslot(i)].v;
  }
  cl.sync();
  if (c == 0 && t == 0) {
    Hand& h = P.ctrl->hand;
    const long long filled = (long long)atomicAdd(&h.qfill, 0ull);
    h.mode = fr == 0 ? 0 : 2;
    h.qs = base;
    h.qe = base + filled;  // == base + fr
    h.qtail = base + filled;
    h.etc = etc;
    h.scout = scout;
    h.nsteps = nsteps;
    h.reached = reached;
    h.lvl = lvl;
    h.swap = H.swap;  // bitmaps untouched
    P.ctrl->num_steps = nsteps;
  }
}

}  // namespace

cudaError_t cluster_configure(int device, int* cluster, int64_t* max_scout) {
  *cluster = 0;
  *max_scout = 0;
  if (getenv("GK_NO_CLUSTER_MODE")) return cudaSuccess;
  cudaError_t e;
  const size_t smem = sizeof(CmShared);
  if ((e = cudaFuncSetAttribute(bfs_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  cudaFuncSetAttribute(bfs_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  int cs_max = 16;
  if (const char* e = getenv("GK_CM_CLUSTER")) cs_max = atoi(e) >= 16 ? 16 : atoi(e) >= 8 ? 8 : 4;  // A/B
  for (int cs = cs_max; cs >= 4; cs /= 2) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kCmBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)bfs_cluster, &cfg) == cudaSuccess && n >= 1) {
      *cluster = cs;
      *max_scout = (int64_t)cs * kCmCap / 2;
      return cudaSuccess;
    }
    cudaGetLastError();
  }
  (void)device;
  return cudaSuccess;
}

cudaError_t cluster_launch(const BfsParams& p, const Hand& h, int cluster, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kCmBlock);
  cfg.dynamicSmemBytes = sizeof(CmShared);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, bfs_cluster, p, h);
}

}  // namespace gk
