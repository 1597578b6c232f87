// gk_persistent.cuh -- device building blocks shared by the persistent
// cooperative kernels (bfs_persistent in gk_bfs_kernel.cu, bc_persistent in
// gk_bc.cu): the shared-memory layout, cache-hinted loads, the grid barrier,
// CTA-wide scans / reductions and per-warp queue appends.  Everything has
// internal linkage (anonymous namespace), so each kernel file compiles its
// own copy.
#pragma once

#include <cooperative_groups.h>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef GK_BITMAP_HINTS
#define GK_BITMAP_HINTS 1  // evict_last on bitmap loads
#endif
#ifndef GK_PARENT_HINTS
#define GK_PARENT_HINTS 1  // evict_first on random parent stores
#endif
#ifndef GK_LD_CLOBBER
#define GK_LD_CLOBBER 1  // "memory" clobber on the bitmap loads (A/B switch)
#endif
#if GK_LD_CLOBBER
#define GK_MEMCLOB : "memory"
#else
#define GK_MEMCLOB
#endif
#ifndef GK_FRONT_NC
#define GK_FRONT_NC 0  // A/B only: the non-coherent path for front loads (not legal for kernel-written data)
#endif
#ifndef GK_STREAM_HINTS
#define GK_STREAM_HINTS 1  // evict_first on top-down adjacency loads
#endif
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
    uint32_t bu_acc[kWarps][32];     // bottom-up: per-warp next bits of a task
    double bc_sig[kBlock];           // Brandes forward: sigma of the tile's frontier vertices
  };
  long long red[kWarps + 2];
  unsigned long long bcast[4];
  unsigned long long snap[kSlots];  // counter set of the phase the last grid_sync ended
  unsigned own_cnt[kOwnWin];        // td_own: claims logged per window
  int ok;
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
// CTA index / count within this traversal's rank (ranks sharing one launch
// take consecutive runs of P.cpr CTAs).
__device__ __forceinline__ int cta_id(const BfsParams& P) { return P.cpr ? (int)(blockIdx.x % P.cpr) : (int)blockIdx.x; }
__device__ __forceinline__ int cta_count(const BfsParams& P) { return P.cpr ? P.cpr : (int)gridDim.x; }
// Counter set of phase ph for this rank's own work (see global_slot).
__device__ __forceinline__ unsigned long long* rset(const BfsParams& P, unsigned ph) {
  return P.rslot ? P.ctrl->rcnt[ph & 3][P.rslot - 1] : P.ctrl->cnt[ph & 3];
}
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
#if GK_BITMAP_HINTS
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()) GK_MEMCLOB);
#else
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) GK_MEMCLOB);
#endif
  return v;
}
// Visited word for a claim pre-check: may be served stale from L1 (bits
// are only ever set, so a stale 0 merely costs the atomic that follows).
__device__ __forceinline__ uint32_t ld_bits_l1(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.ca.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()) GK_MEMCLOB);
  return v;
}
// Front bitmap word within a bottom-up phase: no thread writes it during the
// phase, but the same kernel wrote it in an earlier one, so this is a weak
// L1-cacheable load (not ld.global.nc, which PTX defines only for data that
// is read-only for the kernel's whole lifetime).  Ordering: the grid
// barrier's release-add / acquire-load pair (thread 0) plus bar.sync make
// the earlier phase's stores visible; the acquire invalidates this SM's L1,
// so no line cached before the barrier is served after it.  volatile +
// "memory" keeps the compiler from moving the load across the barrier.
__device__ __forceinline__ uint32_t ld_front(const uint32_t* p) {
  uint32_t v;
#if GK_FRONT_NC
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()) GK_MEMCLOB);
#elif GK_BITMAP_HINTS
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()) GK_MEMCLOB);
#else
  asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p) GK_MEMCLOB);
#endif
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
#if GK_STREAM_HINTS
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_first()));
#else
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
  return v;
}
// Random parent writes: do not let them displace the bitmaps in L2.
__device__ __forceinline__ void st_parent(int32_t* p, int32_t v) {
#if GK_PARENT_HINTS
  asm volatile("st.global.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(policy_evict_first()) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ int64_t ld_off(const int64_t* p) { return __ldg(p); }
// Offset v of the CSR: from the compact form when the graph has one (4
// bytes per vertex instead of 8 -- the bottom-up sweep reads one per pending
// vertex), else the int64 array base (out_off or in_off; they are the same
// array whenever off32 exists).
// GK_OFFMODE fixes the choice at compile time for the grid kernel's two
// instantiations (the run-time test costs registers in its hot loops).
#ifndef GK_OFFMODE
#define GK_OFFMODE 2  // 0: int64 offsets, 1: compact offsets (P.off32 set), 2: chosen at run time
#endif
__device__ __forceinline__ int64_t offv(const BfsParams& P, const int64_t* base, int64_t v) {
  if (GK_OFFMODE == 1 || (GK_OFFMODE == 2 && P.off32))
    return (int64_t)__ldg(P.off32 + v) + ((int64_t)(v >= (int64_t)P.off_hi[0]) << 32);
  return __ldg(base + v);
}

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
    const volatile unsigned long long* rs = rset(P, ph);
#pragma unroll
    for (int i = 0; i < kSlots; i++) s.snap[i] = global_slot(i) ? cs[i] : rs[i];
    if (blockIdx.x == 0) {  // recycle the counter set two phases ahead; trace
      unsigned long long* z = c->cnt[(ph + 3) & 3];
#pragma unroll
      for (int i = 0; i < kSlots; i++) z[i] = 0;
      if (P.cpr)
        for (int i = 0; i < kMaxRanks * kSlots; i++) (&c->rcnt[(ph + 3) & 3][0][0])[i] = 0;
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
  return QApp{base, &rset(P, ph)[kAppend]};
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

}  // namespace
}  // namespace gk
