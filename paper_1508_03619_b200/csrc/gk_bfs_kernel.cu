// gk_bfs_kernel.cu -- direction-optimizing BFS as ONE persistent kernel.
//
// Restates gapkit::Bfs (proj/include/gapkit/kernels/bfs.hpp:117-177) for
// sm_100a.  The whole level loop runs on the device: one cooperative launch
// of 148 x k CTAs, grid barriers between phases, and the reference's
// alpha/beta direction decision (bfs.hpp:143-144, 153-154, 156, 158)
// evaluated redundantly by every thread from counters reduced in L2.  No
// host round trip per level, so high-diameter graphs pay ~a grid barrier
// per level instead of a launch + sync.
//
// Phases (each ends at a grid barrier):
//   init      parent[:] = -1, visited[:] = 0, parent[src] = src, queue = [src]
//             (replaces the degree-encoding init bfs.hpp:126-132: the
//             claim test uses a 1-bit visited map in L2 instead of the
//             parent sign, and the claimed vertex's degree -- what the
//             encoding carries -- is read from the offsets at claim time;
//             scout = sum(max(deg,1)) is identical to sum(-old) of
//             bfs.hpp:83)
//   TD light  frontier tiles of 512 vertices, CTA-wide scan of degrees,
//             load-balanced edge gather (bfs.hpp:68-91); vertices of degree
//             > chunk are cut into chunk-edge chunks (128..1024 by step size)
//   TD heavy  chunks spread over all warps (hub expansion)
//   q2b       QueueToBitmap (bfs.hpp:93-97)
//   BU        one warp per 32-vertex bitmap word: visited-word skip, per-lane
//             scan of the first 4 in-neighbours, then warp-ballot scans of
//             the remaining lists; the first hit in ascending order is the
//             parent exactly as bfs.hpp:55-60 picks it
//   b2q       BitmapToQueue (bfs.hpp:99-113), CTA-aggregated appends
//   rescan    kTopDownRescan's extra degree pass (bfs.hpp:161-167)
#include <cooperative_groups.h>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kQBuf = 256;         // per-warp queue staging (QueueBuffer analogue)
constexpr int kChunkMax = 1024;    // edges per heavy chunk (large steps)
constexpr int kChunkMin = 128;     // ... and for small steps, so every warp gets a chunk
constexpr long long kTinyStep = 1 << 16;  // top-down steps up to this many edges are latency-first
constexpr long long kTinyFrontier = 32768;  // ... and this many frontier vertices


struct __align__(16) SmemT {
  struct {  // top-down phases
    uint32_t qbuf[kWarps][kQBuf];
    int64_t t_b[kBlock];
    int64_t t_pre[kBlock];
    uint32_t t_u[kBlock];
  } td;
  union {
    uint32_t bu_acc[kWarps][2][32];  // bottom-up: per-warp next/dead bits of a task
    double bc_sig[kBlock];           // Brandes forward: sigma of the tile's frontier vertices
  };
  long long red[kWarps + 2];
  unsigned long long bcast[4];
  unsigned long long snap[kSlots];  // counter set of the phase the last grid_sync ended
  int ok;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// L2 cache policy hints: the bitmaps (visited / front, n/8 bytes each) are
// the only reused working set, the graph arrays stream past them.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Bitmap word, bypassing L1 (other SMs update bitmaps within a phase), kept in L2.
__device__ __forceinline__ uint32_t ld_bits(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}
// Visited word for a claim pre-check: may be served stale from L1 (bits
// are only ever set, so a stale 0 merely costs the atomic that follows).
__device__ __forceinline__ uint32_t ld_bits_l1(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.ca.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}
// Read-only front bitmap word within a bottom-up phase: L1-cacheable, kept in L2.
__device__ __forceinline__ uint32_t ld_front(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}
// Graph data: read-only path, default L2 policy (an evict-first hint made
// bottom-up slower: the next round re-reads the same neighbour sector).
__device__ __forceinline__ uint32_t ld_nb(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Top-down edge lists are read exactly once per step: stream them.
__device__ __forceinline__ uint32_t ld_nb_once(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_first()));
  return v;
}
// Random parent writes: do not let them displace the bitmaps in L2.
__device__ __forceinline__ void st_parent(int32_t* p, int32_t v) {
  asm volatile("st.global.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(policy_evict_first()) : "memory");
}
__device__ __forceinline__ int64_t ld_off(const int64_t* p) { return __ldg(p); }

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid barrier on a monotonic arrival counter: barrier k completes when the
// counter reaches k * gridDim.x.  The release-add publishes this CTA's
// stores (ordered before it by __syncthreads); the acquire spin orders the
// CTA's later loads after every other CTA's stores.  A watchdog turns a hang
// into an error instead of a stuck GPU.  Measured ~1.3 us per barrier at
// 296 CTAs on B200 (tools/bench_mem/barbench.cu).
__device__ bool grid_sync(const BfsParams& P, SmemT& s, unsigned& ph, unsigned char tag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    Ctrl* c = P.ctrl;
    int ok = 1;
    if (blockIdx.x < 2048) c->cta_ph[blockIdx.x] = ph + 1;
    red_release_add(&c->bar_count, 1ull);
    const unsigned long long target = (unsigned long long)(ph + 1) * gridDim.x;
    unsigned spins = 0;
    unsigned long long t0 = 0;
    while (ld_acquire_u64(&c->bar_count) < target) {
      if ((++spins & 255u) == 0) {
        if (*reinterpret_cast<volatile int*>(&c->error) == 2) {
          ok = 0;
          break;
        }
        const unsigned long long now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > P.timeout_ns) {
          atomicExch(&c->error, 2);
          ok = 0;
          break;
        }
      }
    }
    s.ok = ok;
    // One read of the ended phase's counters per CTA, shared through smem
    // (every thread reading them from L2 made a hot spot on one line).
    const volatile unsigned long long* cs = c->cnt[ph & 3];
#pragma unroll
    for (int i = 0; i < kSlots; i++) s.snap[i] = cs[i];
    if (blockIdx.x == 0) {  // recycle the counter set two phases ahead; trace
      unsigned long long* z = c->cnt[(ph + 3) & 3];
#pragma unroll
      for (int i = 0; i < kSlots; i++) z[i] = 0;
      if (ph + 1 < (unsigned)kTraceCap) {
        c->ts[ph + 1] = globaltimer();
        c->tag[ph + 1] = tag;
      }
    }
  }
  __syncthreads();
  ph++;
  // Profiling aid (GK_STOP_AFTER): every CTA leaves after the same barrier.
  return s.ok != 0 && ph < P.stop_after;
}

// Exclusive scan of one int64 per thread across the CTA; *total gets the sum.
__device__ int64_t block_exscan(int64_t x, int64_t* total, SmemT& s) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  int64_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= (unsigned)o) incl += y;
  }
  if (lane == 31) s.red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (unsigned)kWarps ? s.red[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, wi, o);
      if (lane >= (unsigned)o) wi += y;
    }
    if (lane < (unsigned)kWarps) s.red[lane] = wi - w;
    if (lane == kWarps - 1) s.red[kWarps] = wi;
  }
  __syncthreads();
  int64_t r = s.red[warp] + incl - x;
  *total = s.red[kWarps];
  __syncthreads();
  return r;
}

// CTA sum; one atomicAdd into the counter ring by thread 0.
__device__ void block_add(long long x, unsigned long long* dst, SmemT& s) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(kFull, x, o);
  if (lane == 0) s.red[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < kWarps; i++) t += s.red[i];
    if (t) atomicAdd(dst, (unsigned long long)t);
  }
  __syncthreads();
}

// Queue appends of one phase land at base + fetch-add on that phase's ring
// counter; after the barrier every thread advances its copy of the tail by
// the counter (a single live tail would race with the next phase's appends).
struct QApp {
  unsigned long long base;
  unsigned long long* ctr;
};
__device__ __forceinline__ QApp qapp(const BfsParams& P, unsigned ph, unsigned long long base) {
  return QApp{base, &P.ctrl->cnt[ph & 3][kAppend]};
}

// Per-warp staging buffer flushed with one fetch-add (QueueBuffer,
// sliding_queue.hpp:62-86).  Must be called by all 32 lanes.
__device__ __forceinline__ void wq_flush(const BfsParams& P, const QApp& qa, uint32_t* buf, int& qcnt) {
  __syncwarp();
  if (qcnt == 0) return;
  unsigned long long base = 0;
  if (lane_id() == 0) base = qa.base + atomicAdd(qa.ctr, (unsigned long long)qcnt);
  base = __shfl_sync(kFull, base, 0);
  for (int i = lane_id(); i < qcnt; i += 32) P.queue[base + i] = buf[i];
  __syncwarp();
  qcnt = 0;
}

__device__ __forceinline__ void wq_push(const BfsParams& P, const QApp& qa, bool claim, uint32_t v,
                                        uint32_t* buf, int& qcnt) {
  unsigned mask = __ballot_sync(kFull, claim);
  if (!mask) return;
  if (claim) buf[qcnt + __popc(mask & lanemask_lt())] = v;
  qcnt += __popc(mask);
  if (qcnt > kQBuf - 32) wq_flush(P, qa, buf, qcnt);
}

// Claim v for parent u (bfs.hpp:78-84).  The visited word is read from L2
// first so already-visited targets cost no atomic.
__device__ __forceinline__ bool try_claim(const BfsParams& P, uint32_t v) {
  const uint32_t bit = 1u << (v & 31u);
  uint32_t* w = P.visited + (v >> 5);
  if (__ldcg(w) & bit) return false;
  return (atomicOr(w, bit) & bit) == 0;
}

__device__ __forceinline__ void on_claim(const BfsParams& P, uint32_t u, uint32_t v, int lvl,
                                         bool encode, long long& scout) {
  P.parent[v] = (int32_t)u;
  if (P.want_depth) P.depth[v] = lvl + 1;
  if (encode) {
    long long d = P.out_off[v + 1] - P.out_off[v];
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
        o0[k] = P.out_off[v[k]];
        o1[k] = P.out_off[v[k] + 1];
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
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) wq_push(P, qa, c[k], v[k], buf, qcnt);
    return;
  }
  if (kBig) {
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
        st_parent(P.parent + v[k], (int32_t)u[k]);
        atomicOr(nextbm + (v[k] >> 5), 1u << (v[k] & 31u));  // result unused -> RED
      }
    }
    return;
  }
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

// ---- top-down, light vertices + chunk registration ------------------------
template <bool kBig>
__device__ void td_light(const BfsParams& P, SmemT& s, unsigned ph, const QApp& qa, unsigned long long qs,
                         unsigned long long qe, uint32_t* nextbm, int lvl, bool encode,
                         long long& scout, int& qcnt, int tile_sz, int64_t chunk, bool tiny,
                         bool reg = true, uint32_t rlo = 0, uint32_t rhi = 0xffffffffu) {
  uint32_t* buf = s.td.qbuf[threadIdx.x >> 5];
  unsigned long long* cnt = P.ctrl->cnt[ph & 3];
  // First tile of each CTA is static (no atomic on the latency chain of
  // small levels); the rest are handed out dynamically.
  unsigned long long tile = blockIdx.x;
  for (;;) {
    const unsigned long long start = qs + tile * (unsigned long long)tile_sz;
    if (start >= qe) break;
    const unsigned long long i = start + threadIdx.x;
    uint32_t u = 0;
    int64_t b = 0, dl = 0;
    if ((int)threadIdx.x < tile_sz && i < qe) {
      u = __ldcg(P.queue + i);
      b = P.out_off[u];
      const int64_t d = P.out_off[u + 1] - b;
      if (d > chunk) {
        if (reg) {  // range passes after the first reuse the chunk list
          const int64_t nch = (d + chunk - 1) / chunk;
          const unsigned long long base = atomicAdd(&cnt[kChunkCount], (unsigned long long)nch);
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
    const bool more = qs + (unsigned long long)gridDim.x * tile_sz < qe && start + tile_sz < qe;
    if (threadIdx.x == 0 && more) s.bcast[1] = gridDim.x + atomicAdd(&cnt[kTile], 1ull);
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
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
  if (kBig) {
    // 8 edges per lane in flight and the next chunk descriptor prefetched:
    // the hub step is bound by the nb -> bitmap-word dependent latency
    constexpr int kE = 8;
    // first chunk static, later ones claimed dynamically; the next claim and
    // its descriptor load are issued before the current chunk's edges
    unsigned long long* cctr = &P.ctrl->cnt[ph & 3][kChunkNext];
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
            st_parent(P.parent + v[k], (int32_t)ch.u);
            atomicOr(nextbm + (v[k] >> 5), 1u << (v[k] & 31u));
          }
        }
      }
      ch = chn;
      c = cn;
    }
    return;
  }
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
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
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
    const int cnt = __popc(cl);
    count += cnt;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const int excl = incl - cnt;
    const int total = __shfl_sync(kFull, incl, 31);
    for (int base = 0; base < total; base += 128) {
      int64_t o0[4], o1[4];
      int64_t v[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int c = base + k * 32 + (int)lane;
        int lo = 0;  // word holding the c-th claim: last lane with excl <= c
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int e = __shfl_sync(kFull, excl, lo + step);
          if (e <= c) lo += step;
        }
        const uint32_t m = __shfl_sync(kFull, cl, lo);
        const int ex = __shfl_sync(kFull, excl, lo);
        v[k] = -1;
        o0[k] = o1[k] = 0;
        if (c < total) {
          v[k] = (w0 + lo) * 32 + (int)__fns(m, 0, c - ex + 1);
          o0[k] = __ldg(P.out_off + v[k]);
          o1[k] = __ldg(P.out_off + v[k] + 1);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (v[k] < 0) continue;
        const long long d = o1[k] - o0[k];
        scout += encode ? (d ? d : 1) : 1;
        if (P.want_depth) P.depth[v[k]] = lvl + 1;
      }
    }
    nx = nx_n;
    vis = vis_n;
  }
}

// ---- bottom-up sweep (bfs.hpp:47-66) ---------------------------------------
// A warp takes a task of 32 consecutive bitmap words (1024 vertices): lane l
// loads word l and the task's unvisited vertices are numbered by a warp
// prefix sum.  Every lane keeps kBuSlots vertices in flight and refills a slot
// (select-the-c-th-pending-vertex: shuffle binary search + __fns) as soon as
// its vertex resolves, so one slow list never idles the other lanes.  Per
// round a slot tests the next kPerRound in-neighbours of its vertex: round 1
// reads the vertex's head (its first kHead in-neighbours, a dense 16-byte
// record per vertex, so the sweep streams it in vertex order instead of
// paying one random in_nb sector per vertex), later rounds continue in
// in_nb.  After kLaneRounds rounds a still-unresolved vertex is deferred to
// the long list, scanned after the sweep by whole warps with a ballot per 32
// neighbours.  The chosen parent is the first in-neighbour (ascending) whose
// front bit is set, as in bfs.hpp:55-60.  Results are OR-ed into per-warp
// shared-memory words and written back once per task.  Vertices without
// in-edges never appear: visited starts as the graph's dead bitmap.
constexpr int kBuSlots = 2;
constexpr int kPerRound = 4;    // in-neighbours tested per slot per round
constexpr int kLaneRounds = 8;  // rounds before a list is deferred to the long list
static_assert(kHead <= kPerRound, "a head round tests one head record");

// front is either the global bitmap or its shared-memory copy (small graphs).
template <bool kSmem>
__device__ __forceinline__ bool front_bit(const uint32_t* front, uint32_t u) {
  const uint32_t w = kSmem ? front[u >> 5] : ld_front(front + (u >> 5));
  return (w >> (u & 31u)) & 1u;
}

template <bool kSmem>
__device__ void bu_step(const BfsParams& P, SmemT& s, unsigned ph, const uint32_t* front, uint32_t* next,
                        int lvl, unsigned long long long_base, int tw_log, long long& awake) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* acc_n = s.bu_acc[warp][0];
  uint32_t* acc_d = s.bu_acc[warp][1];
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
  // A task is 2^tw_log consecutive words (<= 32): small graphs use small
  // tasks so every warp gets work.
  const int tw = 1 << tw_log;
  const long long ntasks = (P.w32 + tw - 1) >> tw_log;
  // First task static, later ones claimed dynamically (per-task work varies
  // with the pending density and list lengths; a static stride left warps
  // idle at the phase's barrier).  The next claim is issued when a task
  // starts, so its round trip hides behind the task.
  unsigned long long* tctr = &P.ctrl->cnt[ph & 3][kTile];
  for (long long t = gw; t < ntasks;) {
    long long tnext = 0;
    if (lane == 0) tnext = nw + (long long)atomicAdd(tctr, 1ull);
    const long long tbase = t << tw_log;
    const long long w = tbase + lane;
    uint32_t vis = 0xffffffffu, pad = 0u, live = 0u, hb = 0u;
    if ((int)lane < tw && w < P.w32) {
      vis = ld_bits(P.visited + w);
      live = ~__ldg(P.dead + w);
      hb = __ldg(P.hbase + w);
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
    acc_n[lane] = 0u;
    acc_d[lane] = 0u;
    __syncwarp();
    int next_c = 0;
    uint32_t v[kBuSlots], d[kBuSlots], rounds[kBuSlots];
    int64_t b[kBuSlots];
    int st[kBuSlots];  // 0 empty, 1 head round, 2 in_nb rounds
#pragma unroll
    for (int k = 0; k < kBuSlots; k++) {
      st[k] = 0;
      v[k] = d[k] = rounds[k] = 0;
      b[k] = 0;
    }
    for (;;) {
      // refill empty slots with the next pending vertices of the task
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        const bool need = st[k] == 0;
        const unsigned nm = __ballot_sync(kFull, need);
        const int c = next_c + __popc(nm & lanemask_lt());
        next_c += __popc(nm);
        int lo = 0;  // word holding the c-th pending vertex: last lane with excl <= c
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int e = __shfl_sync(kFull, excl, lo + step);
          if (e <= c) lo += step;
        }
        const uint32_t m = __shfl_sync(kFull, pm, lo);
        const int ex = __shfl_sync(kFull, excl, lo);
        const uint32_t lv = __shfl_sync(kFull, live, lo);
        const uint32_t hbl = __shfl_sync(kFull, hb, lo);
        if (need && c < total) {
          const uint32_t bit = __fns(m, 0, c - ex + 1);
          v[k] = (uint32_t)((tbase + lo) * 32 + (int)bit);
          b[k] = (int64_t)hbl + __popc(lv & ((1u << bit) - 1u));  // head record (head rounds)
          rounds[k] = 0;
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
      // Round 1 of a vertex reads its head (dense, vertex order); later
      // rounds continue in in_nb after the head.
      uint32_t u[kBuSlots][kPerRound];
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        if (st[k] == 1) {
          head_unpack(__ldg(P.head + b[k]), u[k]);
        } else {
#pragma unroll
          for (int j = 0; j < kPerRound; j++)
            u[k][j] = (st[k] && d[k] > (uint32_t)j) ? ld_nb(P.in_nb + b[k] + j) : kNoVertex;
        }
      }
#pragma unroll
      for (int k = 0; k < kBuSlots; k++) {
        if (!st[k]) continue;
        bool hit = false;
        uint32_t par = 0;
#pragma unroll
        for (int j = 0; j < kPerRound; j++) {
          if (!hit && u[k][j] != kNoVertex && front_bit<kSmem>(front, u[k][j])) {
            hit = true;
            par = u[k][j];
          }
        }
        if (hit) {
          P.parent[v[k]] = (int32_t)par;
          if (P.want_depth) P.depth[v[k]] = lvl + 1;
          atomicOr(&acc_n[(v[k] >> 5) - tbase], 1u << (v[k] & 31u));
          st[k] = 0;
        } else if (st[k] == 1) {
          if (u[k][0] == kNoVertex) {  // no in-edges: never reachable; skip it from now on
            atomicOr(&acc_d[(v[k] >> 5) - tbase], 1u << (v[k] & 31u));
            st[k] = 0;
          } else if (u[k][kHead - 1] == kNoVertex) {
            st[k] = 0;  // the list ended inside the head: not reached at this level
          } else {
            b[k] = ld_off(P.in_off + v[k]) + kHead;
            d[k] = (uint32_t)(ld_off(P.in_off + v[k] + 1) - b[k]);
            rounds[k] = 1;
            st[k] = d[k] ? 2 : 0;
          }
        } else {
          const uint32_t tk = d[k] < (uint32_t)kPerRound ? d[k] : (uint32_t)kPerRound;
          b[k] += tk;
          d[k] -= tk;
          if (d[k] == 0) {
            st[k] = 0;  // exhausted: not reached at this level
          } else if (++rounds[k] >= kLaneRounds) {
            P.queue[long_base + atomicAdd(&P.ctrl->cnt[ph & 3][kLongCount], 1ull)] = v[k];
            st[k] = 0;
          }
        }
      }
    }
    __syncwarp();
    if ((int)lane < tw && w < P.w32) {
      const uint32_t nbits = acc_n[lane], dbits = acc_d[lane];
      next[w] = nbits;
      if (nbits | dbits) P.visited[w] = vis | nbits | dbits;
      awake += __popc(nbits);
    }
    __syncwarp();
    t = __shfl_sync(kFull, tnext, 0);
  }
}

// Long in-lists deferred by bu_step: one warp per vertex, ballot over 32
// neighbours at a time, resuming after the head and the kLaneRounds-1
// in_nb rounds bu_step tested.
template <bool kSmem>
__device__ void bu_long(const BfsParams& P, const uint32_t* front, uint32_t* next,
                        unsigned long long base, unsigned long long count, int lvl, long long& awake) {
  const unsigned lane = lane_id();
  const long long gw = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kBlock) >> 5;
  for (long long i = gw; i < (long long)count; i += nw) {
    const uint32_t v = __ldcg(P.queue + base + i);
    const int64_t le = P.in_off[v + 1];
    for (int64_t j = P.in_off[v] + kHead + kPerRound * (kLaneRounds - 1); j < le; j += 32) {
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
        }
        break;
      }
    }
  }
}

// ---- BitmapToQueue (bfs.hpp:99-113) ----------------------------------------
__device__ void b2q(const BfsParams& P, const QApp& qa, const uint32_t* front, SmemT& s) {
  for (long long base = (long long)blockIdx.x * kBlock; base < P.w32;
       base += (long long)gridDim.x * kBlock) {
    const long long w = base + threadIdx.x;
    uint32_t word = w < P.w32 ? __ldcg(front + w) : 0u;
    int64_t tot;
    const int64_t pre = block_exscan(__popc(word), &tot, s);
    if (tot == 0) continue;
    if (threadIdx.x == 0) s.bcast[0] = qa.base + atomicAdd(qa.ctr, (unsigned long long)tot);
    __syncthreads();
    unsigned long long q = s.bcast[0] + pre;
    while (word) {
      const int bp = __ffs(word) - 1;
      word &= word - 1;
      P.queue[q++] = (uint32_t)(w * 32 + bp);
    }
    __syncthreads();
  }
}

__device__ void log_step(const BfsParams& P, long long idx, int dir, long long frontier,
                         long long result, long long etc) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && idx < P.step_cap) {
    gk_step st;
    st.dir = dir;
    st.pad = 0;
    st.frontier = frontier;
    st.result = result;
    st.edges_to_check = etc;
    P.steps[idx] = st;
  }
}

__global__ void __launch_bounds__(kBlock, 2) bfs_persistent(BfsParams P) {
  extern __shared__ uint4 dyn_smem[];
  __shared__ SmemT s;
  unsigned ph = 0;
  const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long gthreads = (long long)gridDim.x * kBlock;
  const uint32_t src = P.src;

  // ---- init (timed; replaces bfs.hpp:126-138) ----
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->ts[0] = globaltimer();
  {
    const long long n4 = P.n >> 2;
    int4* p4 = reinterpret_cast<int4*>(P.parent);
    int4* d4 = reinterpret_cast<int4*>(P.depth);
    const int4 m1 = make_int4(-1, -1, -1, -1);
#pragma unroll 4
    for (long long i = gtid; i < n4; i += gthreads) {
      p4[i] = m1;
      if (P.want_depth) d4[i] = m1;
    }
    for (long long i = (n4 << 2) + gtid; i < P.n; i += gthreads) {
      P.parent[i] = -1;
      if (P.want_depth) P.depth[i] = -1;
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
  if (!grid_sync(P, s, ph, kTagInit)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // bfs.hpp:132-136
    P.parent[src] = (int32_t)src;
    if (P.want_depth) P.depth[src] = 0;
    P.visited[src >> 5] |= 1u << (src & 31u);
    P.queue[0] = src;
  }
  if (!grid_sync(P, s, ph, kTagInit)) return;

  const bool encode = P.strategy != GK_BFS_TOP_DOWN_RESCAN;
  unsigned long long qs = 0, qe = 1;
  unsigned long long qtail = 1;  // queue entries written so far (uniform)
  long long etc = P.m;                                  // bfs.hpp:139
  long long scout = P.out_off[src + 1] - P.out_off[src];  // bfs.hpp:140
  long long nsteps = 0;
  int lvl = 0;
  int qcnt = 0;
  bool front_ready = false;  // frontg holds exactly the current frontier
  bool queue_stale = false;  // the current frontier's queue window is not written yet
  uint32_t* frontg = P.bm0;
  uint32_t* nextg = P.bm1;
  uint32_t* sfront = reinterpret_cast<uint32_t*>(dyn_smem);
  const long long nwarps = gthreads >> 5;
  int bu_tw_log = 5;  // bottom-up task = 32 words unless that leaves warps idle
  while (bu_tw_log > 0 && ((P.w32 + (1 << bu_tw_log) - 1) >> bu_tw_log) < nwarps) bu_tw_log--;

  while (qe > qs) {
    const bool go_bu = P.strategy == GK_BFS_DIRECTION_OPTIMIZING && scout > etc / P.alpha;
    if (!go_bu && queue_stale) {  // BitmapToQueue for the coming top-down step
      const unsigned bset = ph & 3;
      b2q(P, qapp(P, ph, qtail), frontg, s);
      if (!grid_sync(P, s, ph, kTagB2Q)) return;
      qtail += s.snap[kAppend];
      queue_stale = false;
    }
    if (go_bu) {
      if (!front_ready) {  // QueueToBitmap into a cleared front (bfs.hpp:145)
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
        // long-list scratch: queue slots past the tail are unused during bottom-up
        const unsigned long long lbase = qe;
        if (P.front_in_smem) bu_step<true>(P, s, ph, fr, nextg, lvl, lbase, bu_tw_log, acc);
        else bu_step<false>(P, s, ph, fr, nextg, lvl, lbase, bu_tw_log, acc);
        unsigned set = ph & 3;
        block_add(acc, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagBU)) return;
        const unsigned long long nlong = s.snap[kLongCount];
        long long awake_bu = (long long)s.snap[kSum];
        if (nlong) {
          acc = 0;
          if (P.front_in_smem) bu_long<true>(P, fr, nextg, lbase, nlong, lvl, acc);
          else bu_long<false>(P, fr, nextg, lbase, nlong, lvl, acc);
          set = ph & 3;
          block_add(acc, &P.ctrl->cnt[set][kSum], s);
          if (!grid_sync(P, s, ph, kTagLong)) return;
          awake_bu += (long long)s.snap[kSum];
        }
        awake = awake_bu;
        log_step(P, nsteps++, 'B', old_awake, awake, etc);
        lvl++;
        uint32_t* t = frontg;
        frontg = nextg;
        nextg = t;
      } while (awake >= old_awake || awake > P.n / P.beta);
      const unsigned bset = ph & 3;
      b2q(P, qapp(P, ph, qtail), frontg, s);  // bfs.hpp:155
      if (!grid_sync(P, s, ph, kTagB2Q)) return;
      qtail += s.snap[kAppend];
      qe = qtail;
      scout = 1;  // bfs.hpp:156
      front_ready = true;
    } else {
      etc -= scout;  // bfs.hpp:158
      const long long fsize = (long long)(qe - qs);
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
      if (big) {  // next := visited (see claim4<true>)
        for (long long i = gtid; i < P.w32; i += gthreads) nextg[i] = __ldcg(P.visited + i);
        if (!grid_sync(P, s, ph, kTagZero)) return;
      }
      if (big) {
        // Claims only touch next (n/8 bytes).  When that bitmap is larger
        // than L2 can hold, the step runs in P.td_passes passes over target
        // vertex ranges of P.td_span ids, each pass's slice of next (and of
        // parent) staying L2-resident; the frontier's lists are re-streamed
        // per pass, which HBM does at full bandwidth.
        unsigned long long nch = 0;
        for (int r = 0; r < P.td_passes; r++) {
          const uint32_t rlo = (uint32_t)((int64_t)r * P.td_span);
          const uint32_t rhi = r + 1 == P.td_passes ? 0xffffffffu : (uint32_t)((int64_t)(r + 1) * P.td_span);
          set = ph & 3;
          {
            const QApp qa = qapp(P, ph, qtail);
            td_light<true>(P, s, ph, qa, qs, qe, nextg, lvl, encode, sacc, qcnt, tile_sz, chunk, false, r == 0,
                           rlo, rhi);
          }
          if (!grid_sync(P, s, ph, kTagTD)) return;
          if (r == 0) nch = s.snap[kChunkCount];
          if (nch) {
            const QApp qa = qapp(P, ph, qtail);
            td_heavy<true>(P, s, ph, qa, nch, nextg, lvl, encode, sacc, qcnt, false, rlo, rhi);
            if (!grid_sync(P, s, ph, kTagHeavy)) return;
          }
        }
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
      if (big) {
        long long cacc = 0;
        sacc = 0;
        set = ph & 3;
        td_scout_bits(P, nextg, lvl, encode, sacc, cacc);
        block_add(sacc, &P.ctrl->cnt[set][kSum], s);
        block_add(cacc, &P.ctrl->cnt[set][kCount], s);
        if (!grid_sync(P, s, ph, kTagSweep)) return;
        scout = (long long)s.snap[kSum];
        const unsigned long long claimed = s.snap[kCount];
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
        front_ready = false;
        qs = qe;  // SlideWindow (bfs.hpp:160)
        qe = qtail;
      }
      if (P.strategy == GK_BFS_TOP_DOWN_RESCAN) {  // bfs.hpp:161-167
        long long tot = 0;
        for (unsigned long long i = qs + gtid; i < qe; i += gthreads) {
          const uint32_t u = __ldcg(P.queue + i);
          tot += P.out_off[u + 1] - P.out_off[u];
        }
        set = ph & 3;
        block_add(tot, &P.ctrl->cnt[set][kSum], s);
        if (!grid_sync(P, s, ph, kTagRescan)) return;
        scout = (long long)s.snap[kSum];
      }
      log_step(P, nsteps++, 'T', fsize, scout, etc);
      lvl++;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->num_steps = nsteps;
  // bfs.hpp:171-175's final sweep is unnecessary: unreached slots were
  // written -1 by init and never touched.
}


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
      b = P.out_off[u];
      su = __ldcg(&P.bc_sd[u].x);
      const int64_t d = P.out_off[u + 1] - b;
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
      b = P.out_off[u];
      su = __ldcg(&P.bc_sd[u].x);
      const int64_t d = P.out_off[u + 1] - b;
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
        b = P.in_off[v];
        dl = P.in_off[v + 1] - b;
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
      b = P.in_off[v];
      dl = P.in_off[v + 1] - b;
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
        dsum += P.out_off[u + 1] - P.out_off[u];
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
      unsigned set = ph & 3;
      {
        const QApp qa = qapp(P, ph, qtail);
        bc_forward_light(P, s, ph, qa, qs, qe, lvl, qcnt);
        wq_flush(P, qa, s.td.qbuf[threadIdx.x >> 5], qcnt);
      }
      if (!grid_sync(P, s, ph, kTagTD)) return;
      qtail += s.snap[kAppend];
      const unsigned long long nch = s.snap[kChunkCount];
      if (nch) {
        set = ph & 3;
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
          sum += P.out_off[u + 1] - P.out_off[u];
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

cudaError_t bfs_configure(int device, BfsLaunch* cfg) {
  cudaError_t e;
  int sms = 0, optin = 0, coop = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device))) return e;
  if ((e = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device))) return e;
  if (!coop) return cudaErrorNotSupported;
  cfg->smem_static = sizeof(SmemT);
  // Stage the front bitmap in shared memory when it fits next to the
  // static part at 1 CTA/SM; otherwise it is read through L1/L2.
  const size_t budget = (size_t)optin > cfg->smem_static + 1024 ? optin - cfg->smem_static - 1024 : 0;
  cfg->smem_front_max = budget & ~size_t(15);
  if ((e = cudaFuncSetAttribute(bfs_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)cfg->smem_front_max)))
    return e;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_persistent, kBlock, 0))) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  cfg->grid = sms * occ;
  cfg->block = kBlock;
  return cudaSuccess;
}

cudaError_t bfs_launch(const BfsParams& p, const BfsLaunch& cfg, cudaStream_t st) {
  size_t dyn = 0;
  int grid = cfg.grid;
  if (p.front_in_smem) {
    dyn = ((size_t)p.w32 * 4 + 15) & ~size_t(15);
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bfs_persistent, kBlock, dyn);
    if (e) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    grid = sms * occ;
  }
  BfsParams local = p;
  void* args[] = {&local};
  return cudaLaunchCooperativeKernel((const void*)bfs_persistent, dim3(grid), dim3(cfg.block), args,
                                     dyn, st);
}

cudaError_t bc_launch(const BfsParams& p, int device, cudaStream_t st) {
  cudaError_t e;
  int sms = 0, occ = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bc_persistent, kBlock, 0))) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
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
