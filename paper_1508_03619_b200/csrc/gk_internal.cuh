// gk_internal.cuh -- shared device/host internals of libgk_bfs.so.
//
// Layout in HBM (one gk_graph per device):
//   graph     : out_off int64[n+1], out_nb uint32[m]; in_* alias out_* when
//               undirected (graph.hpp:64-67), separate arrays when directed;
//               dead uint32[ceil(n/32)] + live: the in-degree-0 vertices, a
//               graph property read by every traversal kernel (BFS and
//               Brandes seed their visited maps with it).
//   per-trial : parent int32[n]           -- the result (ParentArray)
//   scratch     visited/bm0/bm1 uint32[ceil(n/32)] -- 1 bit per vertex
//               queue uint32[n+1]        -- sliding frontier queue
//                                           (sliding_queue.hpp:24-57)
//               chunks                   -- heavy-vertex edge chunks
//               own_list / own_stage     -- owned-range hub expansion
//               ctrl, step log           -- grid barrier, counter ring, trace
//   Everything per-trial is allocated from the graph's stream-ordered pool
//   and initialised inside the timed region of each trial, and freed at its
//   end (GAP rule: only the graph is reused between trials).
#ifndef GK_INTERNAL_CUH_
#define GK_INTERNAL_CUH_

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/gk_bfs.h"

namespace gk {

// Counter ring: a phase (the interval between two grid barriers) that
// accumulates counters uses set ph&3; set (ph+2)&3 is zeroed by CTA 0
// during phase ph (its last reader finished before barrier ph).
// kAppend: queue entries appended during the phase (appends of a phase go
// to tail + fetch-add on it; one live tail would race with the next phase's
// appends).  kLongCount: bottom-up vertices deferred to the long list.
constexpr int kTraceCap = 512;
enum PhaseTag : unsigned char { kTagInit = 'I', kTagTD = 'T', kTagHeavy = 'H', kTagZero = 'Z', kTagQ2B = 'Q',
                                kTagBU = 'B', kTagB2Q = 'C', kTagRescan = 'R', kTagSweep = 'S', kTagLong = 'L',
                                kTagBcBack = 'D', kTagBcChunk = 'E', kTagBcScore = 'F', kTagOwn = 'O', kTagPull = 'P' };
enum CounterSlot { kSum = 0, kTile = 1, kChunkCount = 2, kChunkNext = 3, kAppend = 4, kLongCount = 5, kCount = 6,
                   kOwnCount = 7, kWork = 8, kSlots = 10 };
// kSum, kCount and kWork are traversal-wide totals (kWork: hubs, heavy
// chunks and long lists registered -- the sharded kernel skips a phase no
// rank has work for); the other slots count work of one rank (tiles,
// chunks, queue appends, long lists).  Ranks that share one
// launch (the sharded traversal's single-device emulation) keep those in
// Ctrl::rcnt; ranks on separate devices in their own Ctrl.
__host__ __device__ constexpr bool global_slot(int k) { return k == kSum || k == kCount || k == kWork; }
constexpr int kMaxRanks = 8;

// Hand-off between the grid kernel and the cluster kernel (long chains of
// tiny top-down levels, gk_bfs_cluster.cu): where the traversal stands.
struct Hand {
  long long mode;  // 0 finished, 1 continue in the cluster kernel, 2 continue in the grid kernel
  long long qs, qe, qtail;  // the frontier's queue window, queue entries written so far
  long long etc, scout, nsteps, reached, lvl;
  unsigned long long qfill;  // cluster kernel: entries appended after qtail (overflow, exit)
  long long swap;            // grid kernel: front/next bitmaps swapped (frontg == bm1)
  long long pad;
};

struct Ctrl {
  // ---- cleared before every launch (kCtrlClear bytes) ----
  Hand hand;
  unsigned long long bar_count;  // monotonic grid-barrier arrivals
  int error;
  int pad0;
  long long num_steps;
  long long pad1;
  unsigned long long cnt[4][kSlots];
  unsigned long long rcnt[4][kMaxRanks][kSlots];  // per-rank slots when ranks share a launch
  unsigned long long xsnap[kSlots];  // sharded, multi-device: traversal-wide totals of the last cross-rank barrier
  unsigned long long xsyncs;         // sharded, multi-device: cross-rank barriers this traversal passed
  unsigned long long pad2;
  // Trace: tag[i] names the phase that grid barrier i ended (see PhaseTag),
  // 0 past the last one.
  unsigned char tag[kTraceCap];
  // ---- written before read ----
  // globaltimer at kernel start (ts[0]) and at the release of each of the
  // first kTraceCap-1 grid barriers.
  unsigned long long ts[kTraceCap];
  unsigned int cta_ph[2048];  // per-CTA barrier count (watchdog diagnostics; CTAs < grid)
};
constexpr size_t kCtrlClear = offsetof(Ctrl, ts);
constexpr size_t kCtrlPeek = offsetof(Ctrl, num_steps);  // hand, bar_count, error

static_assert(sizeof(Ctrl) % 16 == 0 && kCtrlClear % 16 == 0, "control blocks are cleared with 16-byte stores");

struct Chunk {
  uint32_t u;
  uint32_t len;
  int64_t start;
};

constexpr uint32_t kNoVertex = 0xffffffffu;
// Neighbour arrays are allocated with this many bytes past the last arc, so
// a 32-byte-aligned sector load covering the last arcs stays inside the
// allocation.
constexpr size_t kNbPad = 32;

// Owned-range hub expansion (large top-down steps): CTA r owns target ids
// [r*span, (r+1)*span) (span = own_span_w*32) and stages that slice of the
// next bitmap in shared memory.  The step's hubs (frontier vertices of
// out-degree >= own_dmin) are listed; each CTA finds the run of every hub's
// ascending out-list that falls in its range by an interpolation search
// inside the trial (no per-graph table).  Claims are logged per window of
// 2^own_win_log ids (kOwnWin windows per range) in own_stage and their
// parents written window by window in vertex order.
constexpr int kOwnWin = 64;  // windows per owned range, at most
struct OwnEnt {
  uint32_t u;
  uint32_t deg;   // out-degree (< 2^32)
  int64_t base;   // out_off[u]
};

struct BfsParams {
  int64_t n;
  int64_t m;
  int64_t w32;  // ceil(n/32)
  const int64_t* out_off;
  const uint32_t* out_nb;
  const int64_t* in_off;
  const uint32_t* in_nb;
  uint32_t src;
  int32_t strategy;
  int64_t alpha;
  int64_t beta;
  int32_t want_depth;
  int32_t front_in_smem;
  int32_t parent_preset;  // parent already holds -1 everywhere (cleared by a memset in the launch)
  int64_t bitmap_td_min;  // scout above which a top-down step is 'large'
  int32_t* parent;
  int32_t* depth;
  uint32_t* visited;
  uint32_t* bm0;
  uint32_t* bm1;
  // graph: the offsets' compact form (undirected graphs up to 2^28 vertices
  // and 2^33 arcs, else null): off[v] = off32[v] + 2^32 * (v >= off_hi[0]),
  // off_hi[0] = first vertex whose offset is >= 2^32 (0xffffffff: none)
  const uint32_t* off32;
  uint32_t off_hi[1];
  const uint32_t* dead;  // graph: in-degree-0 vertices (+ ids >= n), never reachable
  int64_t live;          // graph: vertices with in-edges (not dead)
  uint32_t* queue;
  Chunk* chunks;
  int64_t chunk_cap;
  Ctrl* ctrl;
  gk_step* steps;
  int64_t step_cap;
  unsigned long long timeout_ns;
  unsigned stop_after;  // leave after this many grid barriers (profiling only)
  OwnEnt* own_list;           // the step's hubs (null: owned-range expansion off)
  int64_t own_cap;            // capacity of own_list
  uint2* own_stage;           // [R][windows][2^own_win_log] logged claims {id - window start, parent}
  int32_t own_r;              // ranges = CTAs of the launch
  int32_t own_span_w;         // bitmap words per range (multiple of 4)
  int32_t own_win_log;        // ids per claim-log window = 2^own_win_log <= own_span_w
  int64_t own_dmin;           // out-degree that counts as a hub
  int32_t bu_tw_log_max;  // bottom-up task = 2^this bitmap words (5 unless overridden for A/B)
  // Sharded traversal (gk_bfs_sharded.cu); zero for a single-device traversal.
  int32_t cpr;          // CTAs per rank when several ranks share one launch (emulation), else 0
  int32_t rslot;        // 1 + this rank's slot in Ctrl::rcnt when ranks share a launch, else 0
  int32_t sharded;      // bitmap top-down claims store parents to the target's owner (shard_parent)
  int64_t shard_block;  // vertices per rank
  uint32_t shard_recip; // ceil(2^32 / shard_block)
  int32_t* shard_parent[kMaxRanks];  // per rank: parent array shifted so [v] is owned v's slot (peer-mapped)
  int64_t w_lo, w_hi;   // owned bitmap words [w_lo, w_hi) (0, w32 unsharded)
  // Cluster mode for long chains of tiny top-down levels (gk_bfs_cluster.cu)
  int32_t cm_ok;         // the cluster kernel is available for this traversal
  int32_t resume;        // this launch continues a traversal from rs (skip init)
  int64_t cm_max_scout;  // a top-down step stays in cluster mode while scout <= this
  Hand rs;               // resume state
  int32_t td_passes;    // large top-down steps: target-range passes (1 when next fits L2)
  int64_t td_span;      // ids per pass (multiple of 32)
  // Brandes (betweenness.hpp:38-80), bc_persistent only
  double2* bc_sd;       // per vertex {shortest-path count sigma, dependency delta}
  uint32_t* bc_succ;    // one bit per stored arc: shortest-path successor edge
  float* bc_scores;     // accumulated over sources
  int64_t* bc_bounds;   // level d = queue[bounds[d], bounds[d+1]) (low 56 bits); bits 56..63 = 1 +
                        // index of the level's bitmap in bc_lv when it was found by a pull step
  uint32_t* bc_lv;      // kBcMaxPull level bitmaps of bc_lvw words (pull-found levels)
  int64_t bc_lvw;
  long long* bc_lvdeg;  // [kBcMaxPull] in-arc sum of each pull-found level
  int64_t bc_bounds_cap;
};

constexpr int kBlock = 512;
constexpr int kBcMaxPull = 8;  // Brandes levels found by a pull (bottom-up) step, at most
constexpr int kWarps = kBlock / 32;

// Host-side launch of the persistent traversal kernel.
struct BfsLaunch {
  int grid = 0;
  int block = kBlock;
  size_t smem_static = 0;
  size_t smem_front_max = 0;  // largest front bitmap (bytes) staged in smem
  size_t smem_keep_occ = 0;   // largest dynamic smem that keeps the occupancy of grid
};
cudaError_t bfs_configure(int device, BfsLaunch* cfg);
cudaError_t bfs_launch(const BfsParams& p, const BfsLaunch& cfg, cudaStream_t s);
const void* bfs_resume_fn();  // the grid kernel continuing a handed-back traversal (gk_bfs_resume.cu)
// the same two instantiations reading the compact offsets (gk_bfs_kernel_c.cu, gk_bfs_resume_c.cu)
const void* bfs_fresh_c_fn();
const void* bfs_resume_c_fn();
// ---- sharded traversal (gk_bfs_sharded.cu) --------------
// Rank r owns vertices [lo, hi) (hi - lo = block, a multiple of 1024 so a
// 32-word bottom-up task never straddles two ranks) and the CSR rows of
// those vertices (undirected: in = out).  Bitmaps (visited, front/next,
// claims) are full-n and replicated; parent/depth cover the owned range.
struct ShardView {
  const int64_t* off;  // shifted: off[v] for owned v (row of v - lo)
  const uint32_t* off32;  // shifted compact form of off (BfsParams::off32), or null
  uint32_t off_hi;        // global id of the first owned vertex whose offset is >= 2^32
  const uint32_t* nb;  // neighbour ids are global
  int32_t* parent;     // shifted like off; a registered buffer peers map (remote claims store here)
  int32_t* depth;      // shifted, or null
  uint32_t* queue;     // owned frontier windows + long-list scratch, 2*(hi-lo)+64
  OwnEnt* own_list;    // owned-range hub expansion of this rank's hubs (null: off)
  uint2* own_stage;
  int64_t own_cap;
  Chunk* chunks;
  int64_t chunk_cap;
  uint32_t* bm[4];     // full-n bitmaps: visited, front/next pair, claims
  const uint32_t* dead;  // full-n, replicated graph layout
  int64_t lo, hi;
};
// Cross-rank barrier and counter reduction of separate launches (one per
// device); lives on rank 0, the others map it.
struct XCtrl {
  unsigned long long bar;
  int error;
  int pad;
  unsigned long long cnt[4][kSlots];
};
struct ShardTab {
  int32_t nranks;
  int32_t emulated;  // 1: all ranks in this one launch, cpr CTAs each (one device)
  int32_t rank;      // this launch's rank (emulated == 0)
  int32_t force_x;   // test hook: the multi-device barrier protocol even for one rank
  int64_t m_total;   // arcs of the whole graph (edges_to_check, bfs.hpp:139)
  int64_t block;     // vertices per rank
  int64_t live_total;
  ShardView v[kMaxRanks];  // peers: only bm[] is dereferenced (peer-mapped in multi-device runs)
  XCtrl* x;          // multi-device only
  unsigned long long xbase;  // multi-device: cross-rank barriers completed by earlier traversals
};
cudaError_t shard_configure(int device, BfsLaunch* cfg);
// Cluster kernel: *cluster = CTAs per cluster (0: unavailable), *max_scout =
// the largest step it takes.
cudaError_t cluster_configure(int device, int* cluster, int64_t* max_scout);
cudaError_t cluster_launch(const BfsParams& p, const Hand& h, int cluster, cudaStream_t s);
// Small graphs: the whole traversal inside one thread-block cluster (gk_bfs_small.cu).
cudaError_t small_configure(int device, int64_t n, int64_t m, int* cluster);
// Compact offsets: off32[v] = low 32 bits of off[v]; hi[k] = first v with off[v] >= (k+1) 2^32 (gk_aux.cu).
cudaError_t compact_offsets(const int64_t* off, int64_t n, uint32_t* off32, uint32_t* hi, int nhi,
                            cudaStream_t s);
cudaError_t small_launch(const BfsParams& p, int cluster, cudaStream_t s);
cudaError_t shard_launch(const BfsParams& p, const ShardTab& t, int grid, cudaStream_t s);

// One source of Brandes' forward + backward pass (cooperative launch).
cudaError_t bc_launch(const BfsParams& p, int device, cudaStream_t s);
// scores /= max(scores) when the max is > 0 (betweenness.hpp:136-143).
cudaError_t bc_normalize(float* scores, int64_t n, float* scratch_max, cudaStream_t s);

// Graph layout (built with the graph, shared by BFS and Brandes): dead =
// in-degree-0 vertices and ids >= n; *live = vertices with in-edges.
cudaError_t dead_bitmap(const int64_t* in_off, int64_t n, uint32_t* dead, int64_t* live, cudaStream_t s);
// CSR invariants: n rows with offsets monotone from 0 to m, neighbour ids < id_bound.
// *sorted (may be null: not checked) = every list strictly ascending.
cudaError_t validate_csr(const int64_t* off, const uint32_t* nb, int64_t n, int64_t m, int64_t id_bound,
                         bool* offsets_ok, bool* ids_ok, bool* sorted, cudaStream_t s);
// Bytes of p[0..len) that differ from fill, written to *d_out.
cudaError_t canary_count(const void* p, size_t len, unsigned char fill, unsigned long long* d_out, cudaStream_t s);
cudaError_t count_reached(const int32_t* parent, const int64_t* off, int64_t n,
                          unsigned long long* d_out2, cudaStream_t s);
// Compact ParentArray transfer (gk_pack.cu, gk_expand.cpp): words of the
// transfer buffer, the count + scan pass (reached total lands in buf[nblk]),
// the scatter of the reached parents, and the host expansion.
size_t pack_words(int64_t n);
// host_out (mapped pinned, may be NULL): receives {reached total, off[probe]}.
cudaError_t pack_count(const int32_t* parent, int64_t n, uint32_t* buf, uint32_t* cnt, int64_t probe,
                       uint32_t* host_out, cudaStream_t s);
cudaError_t pack_scatter(const int32_t* parent, int64_t n, uint32_t* buf, cudaStream_t s);
void expand_parents(const uint32_t* buf, int64_t n, int32_t* dst, int threads, int64_t first_block);
bool expand_uses_avx512();
cudaError_t verify_bfs(const int64_t* off, const uint32_t* nb, const int32_t* parent, const int32_t* depth,
                       int64_t n, uint32_t src, long long* errs8, cudaStream_t s);
cudaError_t byte_model(const BfsParams& p, const int32_t* depth, const char* dirs,
                       int32_t nsteps, unsigned long long* d_acc, double* b_sec,
                       double* b_use, cudaStream_t s);

// Device graph construction (gk_graph_build.cu).
struct DevCsr {
  int64_t n = 0;   // global vertex count
  int64_t lo = 0;  // rows [lo, hi) are stored; offsets are local to lo
  int64_t hi = 0;
  int64_t m = 0;   // stored arcs
  int64_t* off = nullptr;
  uint32_t* nb = nullptr;
};
cudaError_t build_generated(int kind, int scale, int degree, uint64_t seed, int permute, int64_t klo,
                            int64_t khi, DevCsr* out, std::string* err);
// Serialized-graph cache (gk_sg.cu); return 0 on success, else an error code
// (2 open, 3 bad magic, 4 truncated/io, 5 version, 6 flags, 7-8 alloc, 9 data).
int sg_load(const char* path, int64_t* n, int64_t* m, int* directed, int64_t** off, uint32_t** nb,
            int64_t** in_off, uint32_t** in_nb, std::string* err);
int sg_save(const char* path, int64_t n, int64_t m, int directed, const int64_t* off, const uint32_t* nb,
            const int64_t* in_off, const uint32_t* in_nb, std::string* err);
cudaError_t build_grid(int64_t rows, int64_t cols, double p_delete, double p_diag,
                       uint64_t seed, DevCsr* out, std::string* err);

}  // namespace gk

// Scratch of one traversal (gk_bfs / one gk_bfs_batch trial), carved from
// the graph's memory pool inside the timed region and returned at its end.
struct gk_trial {
  int32_t* parent = nullptr;   // the result; outlives the trial until the next one
  uint32_t* bits = nullptr;    // visited | bm0 | bm1, bits_stride words apart
  size_t bits_stride = 0;
  uint32_t* queue = nullptr;
  gk::Chunk* chunks = nullptr;
  gk::OwnEnt* own_list = nullptr;
  uint2* own_stage = nullptr;
  gk::Ctrl* ctrl = nullptr;
  gk_step* steps = nullptr;
};

struct gk_graph {
  int device = 0;
  int64_t n = 0;
  int64_t m = 0;
  int32_t directed = 0;
  int64_t* out_off = nullptr;
  uint32_t* out_nb = nullptr;
  int64_t* in_off = nullptr;  // == out_off when undirected
  uint32_t* in_nb = nullptr;
  // graph layout shared by the traversal kernels (BFS, Brandes), built with the graph
  uint32_t* dead = nullptr;  // in-degree 0 (never reachable) + ids >= n
  uint32_t* off32 = nullptr;  // compact offsets (BfsParams::off32), undirected graphs <= 2^28 vertices
  uint32_t off_hi[1] = {0xffffffffu};
  int64_t live = 0;          // vertices with in-edges
  // per-trial scratch comes from this pool (stream-ordered, kept warm between
  // trials so an allocation is a pointer bump, not an OS call)
  cudaMemPool_t pool = nullptr;
  int64_t chunk_cap = 0;
  int64_t step_cap = 0;
  bool canary = false;  // GK_CANARY=1: guard zones after every trial buffer (debug)
  int own_r = 0;  // owned-range hub expansion geometry (0: off for this graph)
  int64_t own_span_w = 0, own_dmin = 0, own_cap = 0;
  int own_win_log = 0;
  size_t own_stage_bytes = 0;
  // the last traversal's result, kept for gk_bfs_device_parent / verify / model
  int32_t* parent = nullptr;
  int32_t* depth = nullptr;  // diagnostic depth array (parity / model runs), lazily
  unsigned long long* acc = nullptr;  // aux accumulators
  int32_t keep_depth = 0;
  int32_t depth_valid = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // D2H stream of gk_bfs_batch (created on first use)
  cudaStream_t cstream2 = nullptr;  // second D2H stream (GK_BATCH_SPLIT)
  cudaEvent_t cs2_done = nullptr;
  // pinned staging for copies into pageable host memory (gk_capi.cu copy_out)
  char* stage = nullptr;
  size_t stage_bytes = 0;
  std::vector<cudaEvent_t> stage_ev;
  int* batch_err = nullptr;        // pinned: per-trial kernel error codes of gk_bfs_batch
  bool batch_warm = false;         // the pool holds three trials' blocks (gk_bfs_batch)
  int32_t batch_err_cap = 0;
  std::vector<cudaEvent_t> batch_ev;  // gk_bfs_batch's events, grown on demand
  // gk_bfs_batch's compact ParentArray transfer (gk_pack.cu): two device
  // transfer buffers and two pinned stages (source i uses i & 1), the block
  // counts, the pinned reached total, count-ready / scatter-done events
  uint32_t* pk_dev[2] = {nullptr, nullptr};
  uint32_t* pk_host[2] = {nullptr, nullptr};
  uint32_t* pk_cnt = nullptr;
  uint32_t* pk_total = nullptr;
  cudaEvent_t pk_ev = nullptr;
  cudaEvent_t pk_sc[2] = {nullptr, nullptr};
  cudaEvent_t pk_cp[2] = {nullptr, nullptr};  // compact part landed (the raw head may still be copying)
  int64_t last_d2h_bytes = 0;  // device->host result bytes of the last gk_bfs_batch
  int64_t last_packed = 0;     // sources of the last gk_bfs_batch sent compact
  bool pk_raw = false;         // a result of this graph gained nothing compact: later ones go raw
  cudaEvent_t ev0 = nullptr;
  cudaEvent_t ev1 = nullptr;
  gk::BfsLaunch launch;
  // cluster mode (gk_bfs_cluster.cu): CTAs per cluster (0: off), largest step it takes,
  // pinned copy of the control block's head (hand-off state + error) read between kernels
  long long launches = 0;  // traversal kernels launched (gk_bfs_launches)
  int cm_cluster = 0;
  int small_cluster = 0;  // gk_bfs_small.cu: CTAs of the single-cluster kernel for this graph (0: not used)
  // gk_bfs on a small graph: one CUDA graph per handle holding the trial's
  // allocation node and the cluster kernel (the kernel arguments are set
  // per trial, ahead of the timed region)
  cudaGraph_t sg_graph = nullptr;
  cudaGraphExec_t sg_exec = nullptr;
  cudaGraphNode_t sg_kernel = nullptr;
  gk_trial sg_trial;
  bool sg_failed = false;
  int64_t cm_max_scout = 0;
  bool cm_batch = false;  // gk_bfs_batch checks for hand-offs after every trial (sparse graphs)
  gk::Ctrl* cm_peek = nullptr;
  gk::Ctrl last_ctrl;  // host copy of the last traversal's control block
  int32_t last_valid = 0;
  std::mutex mu;
};

#endif  // GK_INTERNAL_CUH_
