/*
 * gk_bfs.h -- C ABI of the B200-native direction-optimizing BFS.
 *
 * This is the drop-in boundary for the reference's BFS hot path.  The
 * reference (gapkit, header-only C++20) has no plugin registry or FFI: its
 * "operator API" is the function
 *
 *     ParentArray gapkit::Bfs(const CsrGraph& g, NodeId source,
 *                             const BfsOptions& opts = {});
 *                                 (proj/include/gapkit/kernels/bfs.hpp:117-118)
 *
 * plus the CsrGraph it reads (proj/include/gapkit/graph.hpp:26-183).  The
 * entry points below replace that call; the C++ wrapper in
 * paper_1508_03619_b200/host/gapkit/ restores the exact reference
 * signature on top of them.
 *
 * Conventions: plain pointers and sizes only; no entry point throws or
 * aborts; every failure returns a gk_status and leaves a thread-local
 * message for gk_last_error().  There is no CPU fallback: without a CUDA
 * device every compute entry point returns GK_ERR_NO_DEVICE.
 */
#ifndef GK_BFS_H_
#define GK_BFS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_ABI_VERSION 1

#if defined(__GNUC__)
#define GK_API __attribute__((visibility("default")))
#else
#define GK_API
#endif

typedef enum {
  GK_OK = 0,
  GK_ERR_SOURCE_RANGE = 1, /* bfs.hpp:120-121 ConfigError("bfs source out of range") */
  GK_ERR_BAD_PARAM = 2,    /* bfs.hpp:122-123 ConfigError("bfs alpha and beta must be positive") */
  GK_ERR_CUDA = 3,
  GK_ERR_NCCL = 4,
  GK_ERR_OOM = 5,
  GK_ERR_NO_DEVICE = 6,
  GK_ERR_INVALID = 7,      /* malformed graph / null handle / bad generator spec */
  GK_ERR_TIMEOUT = 8,      /* device-side watchdog fired (never expected) */
  GK_ERR_NO_EDGES = 9,     /* source_picker.hpp:27-28 "cannot pick sources: graph has no edges" */
  GK_ERR_LOAD = 10         /* errors.hpp:35-46 LoadError family (bad magic / version / truncated) */
} gk_status;

/* BfsStrategy (bfs.hpp:37) */
typedef enum {
  GK_BFS_DIRECTION_OPTIMIZING = 0,
  GK_BFS_TOP_DOWN_ONLY = 1,
  GK_BFS_TOP_DOWN_RESCAN = 2
} gk_bfs_strategy;

/* Host view of a CsrGraph (graph.hpp:26-45).  For undirected graphs the
 * in_* arrays must be NULL (they alias the out arrays, graph.hpp:64-67). */
typedef struct {
  int64_t num_nodes;
  int32_t directed;
  int32_t reserved;
  const int64_t* out_offsets;    /* n+1, out_offsets[n] = m arcs */
  const uint32_t* out_neighbors; /* m, each list sorted, no dups/self-loops */
  const int64_t* in_offsets;     /* directed only */
  const uint32_t* in_neighbors;  /* directed only */
} gk_csr_view;

/* One executed step of the direction loop (bfs.hpp:142-169). */
typedef struct {
  int32_t dir;            /* 'T' top-down or 'B' bottom-up (the reference's schedule) */
  int32_t pad;            /* how the step ran when not as dir names: 0, 'P' bottom-up step
                             executed as a push, 'U' top-down step executed as a pull, 'K'
                             top-down step run by the cluster kernel (same claimed set and
                             counters either way) */
  int64_t frontier;       /* frontier size entering the step */
  int64_t result;         /* T: scout count after the step; B: awake count */
  int64_t edges_to_check; /* heuristic's unexplored-arc budget */
} gk_step;

typedef struct {
  /* in */
  gk_step* steps;          /* optional caller buffer for the step log */
  int32_t max_steps;       /* capacity of steps */
  int32_t want_counts;     /* fill reached / component_edges (untimed pass) */
  /* out */
  float device_ms;         /* CUDA-event time of the whole trial: pool allocation of the result
                              and all scratch, their initialisation, the traversal kernel,
                              release of the scratch */
  int32_t num_steps;       /* steps executed (may exceed max_steps) */
  int64_t reached;         /* vertices with parent >= 0 */
  int64_t component_edges; /* sum of out-degree over reached / (directed?1:2) */
} gk_bfs_stats;

typedef struct gk_graph gk_graph;

/* Human-readable description of the last failure on this thread. */
GK_API const char* gk_last_error(void);
GK_API int gk_abi_version(void);
/* Number of CUDA devices visible (0 without a GPU). */
GK_API int gk_device_count(void);

/* Upload a host CSR into HBM on `device` (untimed, like the reference's
 * untimed build, benchmark.hpp:29-34).  Host arrays are only borrowed. */
GK_API gk_status gk_graph_upload(const gk_csr_view* csr, int device, gk_graph** out);

/* Generate + build on the device: bit-identical to
 * GenerateKronecker / GenerateUniform (generator.hpp:56-112) followed by the
 * optional seeded ID permutation and BuildCsr(el, false, true)
 * (builder.hpp:54-186).  kind: 0 = Kronecker (A,B,C = .57,.19,.19),
 * 1 = uniform.  scale in [1, 31]. */
GK_API gk_status gk_graph_generate(int kind, int scale, int degree, uint64_t seed,
                            int permute, int device, gk_graph** out);
/* Road-like grid (config 4): rows x cols 4-neighbour grid, each edge
 * deleted with p_delete, per-cell diagonal shortcut with p_diag. */
GK_API gk_status gk_graph_generate_grid(int64_t rows, int64_t cols, double p_delete,
                                 double p_diag, uint64_t seed, int device,
                                 gk_graph** out);
/* Serialized-graph cache: the reference's ".sg"/".wsg"
 * binary layout (io.hpp:328-456), streamed file -> pinned -> HBM without a
 * host copy of the graph; weights are skipped.  Errors follow ReadSerialized:
 * GK_ERR_LOAD with "...not a serialized graph (bad magic)", "...unsupported
 * version N", "...file shorter than its declared arrays"; GK_ERR_INVALID when
 * the file cannot be opened. */
GK_API gk_status gk_graph_load_sg(const char* path, int device, gk_graph** out);
/* WriteSerialized (io.hpp:364-389) of an unweighted graph from HBM. */
GK_API gk_status gk_graph_save_sg(const gk_graph* g, const char* path);
GK_API void gk_graph_free(gk_graph* g);

GK_API gk_status gk_graph_info(const gk_graph* g, int64_t* num_nodes,
                        int64_t* num_arcs, int32_t* directed);
/* Copy the device CSR to host arrays (any may be NULL). */
GK_API gk_status gk_graph_download(const gk_graph* g, int64_t* out_offsets,
                            uint32_t* out_neighbors, int64_t* in_offsets,
                            uint32_t* in_neighbors);

/* PickSources(g, count, seed) (source_picker.hpp:47-54). */
GK_API gk_status gk_pick_sources(const gk_graph* g, int64_t count, uint64_t seed,
                          uint32_t* out);

/* Bfs(g, source, {alpha, beta, strategy}) (bfs.hpp:117-177).
 * parent_out: host array of num_nodes int32 (the reference's ParentArray),
 *             or NULL to leave the result resident in HBM.
 * depth_out:  optional host array of num_nodes int32 BFS depths (-1 =
 *             unreached); requesting it adds depth stores to the kernel.
 * stats:      optional.
 * Calls on one handle are serialized; the graph is never modified. */
GK_API gk_status gk_bfs(gk_graph* g, uint32_t source, int64_t alpha, int64_t beta,
                 int32_t strategy, int32_t* parent_out, int32_t* depth_out,
                 gk_bfs_stats* stats);

/* gk_bfs over count sources (same validation, results and errors) with
 * parents_out[i] (host, ideally pinned; may repeat or be NULL) receiving
 * traversal i's ParentArray.  The copy of result i (on a second stream)
 * overlaps traversal i+1, as the reference harness's trial loop would if it
 * could (benchmark.hpp:178-185); each trial takes its result and scratch
 * from the handle's pool.  device_ms[i] (may be NULL) = CUDA-event time of
 * trial i, as gk_bfs_stats.device_ms. */
GK_API gk_status gk_bfs_batch(gk_graph* g, const uint32_t* sources, int32_t count, int64_t alpha,
                              int64_t beta, int32_t strategy, int32_t* const* parents_out,
                              float* device_ms);

/* Device->host result bytes the last gk_bfs_batch on this handle moved:
 * from 2^22 vertices each ParentArray travels compact (per 1024-vertex block
 * a reached count prefix, the reached bitmap, the reached vertices' parents)
 * and is expanded into the caller's array on host threads; a source whose
 * reached set leaves nothing to save travels raw (n int32).  *packed (may be
 * NULL) = sources sent compact.  GK_BATCH_PACK=0 turns the compact form off. */
GK_API int64_t gk_bfs_batch_d2h_bytes(const gk_graph* g, int64_t* packed);

/* Device pointer to the parent array of the last gk_bfs on this handle
 * (valid until the next call / free). */
GK_API const int32_t* gk_bfs_device_parent(const gk_graph* g);

/* Device pointer to the depth array the last gk_bfs recorded (it must have
 * requested depth_out or gk_bfs_keep_depth), or NULL.  Test hook for the
 * certificate's tamper tests. */
GK_API int32_t* gk_bfs_device_depth(const gk_graph* g);

/* Traversal kernels launched on g so far (grid kernel launches, cluster
   kernel launches and grid-kernel resumptions of gk_bfs / gk_bfs_batch):
   the difference around a timed region is the number of this library's
   kernels it ran.  Memsets and the pool's bookkeeping are not counted. */
GK_API int64_t gk_bfs_launches(const gk_graph* g);

/* Phase trace of the last gk_bfs: ts_ns[0] = kernel start, ts_ns[i] = release
 * of grid barrier i (globaltimer ns) and tags[i] the phase it ended: 'I' init,
 * 'T' top-down, 'H' heavy-vertex chunks, 'Z' front clear, 'Q' queue->bitmap,
 * 'B' bottom-up, 'C' bitmap->queue, 'R' rescan.  Up to 511 barriers. */
GK_API gk_status gk_bfs_trace(const gk_graph* g, uint64_t* ts_ns, char* tags,
                              int32_t cap, int32_t* count);

/* Sector-aware (B_sec) and element-granular (B_use) algorithmic byte model
 * of the last gk_bfs on this handle; that call must have
 * requested depth_out or GK_KEEP_DEPTH via gk_bfs_keep_depth(). */
GK_API gk_status gk_bfs_byte_model(gk_graph* g, const gk_step* steps,
                            int32_t num_steps, double* b_sec, double* b_use);
/* Device-side BFS certificate of the last gk_bfs (which must have recorded
 * depths): checks verify.hpp:62-98's conditions plus "every arc v->w with v
 * reached has w reached at depth <= depth[v]+1", which together prove the
 * depths are exact BFS distances -- at full size, without a serial BFS.
 * errors[0..6] = violation counts (source, unreached-with-parent, parent
 * range, parent depth, missing parent edge, arc reachability, arc level),
 * errors[7] = smallest offending vertex or -1. */
GK_API gk_status gk_bfs_verify(gk_graph* g, uint32_t source, int64_t* errors);
/* Keep depths on the device for subsequent gk_bfs calls (for the model). */
GK_API gk_status gk_bfs_keep_depth(gk_graph* g, int32_t keep);

/* ---- Brandes betweenness, SURVEY.md §8(f)-4 ----------------------------
 * Replaces ScoreArray gapkit::Brandes(const CsrGraph&, span<const NodeId>)
 * (proj/include/gapkit/kernels/betweenness.hpp:84-145).  scores_out (n
 * floats, may be NULL) receives the max-normalised scores.  Errors, in the
 * reference's order: no sources -> GK_ERR_BAD_PARAM "betweenness requires
 * at least one source"; source >= n -> GK_ERR_SOURCE_RANGE "betweenness
 * source out of range"; out-degree 0 -> GK_ERR_BAD_PARAM "betweenness source
 * has zero out-degree".  *device_ms (may be NULL) = CUDA-event time of all
 * sources plus the normalisation. */
GK_API gk_status gk_brandes(gk_graph* g, const uint32_t* sources, int64_t num_sources,
                            float* scores_out, double* device_ms);

/* ---- Sharded (1D-partitioned) traversal, SURVEY.md §8(e) ----------------
 * Rank r of P (P <= 8) owns vertices [r*block, min(n, (r+1)*block)), block =
 * ceil(n/P) rounded up to 1024, and the CSR rows of those vertices (global
 * neighbour ids; undirected graphs).  A traversal is ONE persistent kernel
 * per rank: the level loop of bfs.hpp:139-169 runs on the device, the ranks
 * exchange bitmap slices through peer memory and meet at a device-side
 * cross-rank barrier that reduces the heuristic's counters -- no host round
 * trip per level (gk_bfs_sharded.cu).  Parents: bottom-up as bfs.hpp:55-60
 * (first in-neighbour in the frontier), top-down claims resolved by their
 * owner the same way; depths exact.
 *
 * Wiring, either
 *   - every rank in this process on ONE device: gk_shard_join_local, then
 *     gk_shard_group_bfs on rank 0 runs all ranks in one cooperative launch
 *     (the single-GPU emulation of the multi-device run), or
 *   - one process per device: gk_shard_export on every rank, exchange the
 *     blobs (gk_shard_handle_size() bytes each), gk_shard_connect with all
 *     of them in rank order, a host barrier, gk_shard_gather_dead; then every
 *     rank calls gk_shard_bfs with the same arguments. */
typedef struct gk_shard gk_shard;
GK_API const char* gk_shard_last_error(void);
/* This rank's rows of the device-generated graph (same graph as
 * gk_graph_generate). */
GK_API gk_status gk_shard_generate(int kind, int scale, int degree, uint64_t seed,
                                   int permute, int rank, int nranks, int device,
                                   gk_shard** out);
/* This rank's rows from host arrays: local_offsets has (hi-lo+1) entries
 * starting at 0; neighbours are global ids (undirected graphs). */
GK_API gk_status gk_shard_upload(int64_t num_nodes, int rank, int nranks,
                                 const int64_t* local_offsets,
                                 const uint32_t* neighbors, int device,
                                 gk_shard** out);
GK_API void gk_shard_free(gk_shard* s);
GK_API gk_status gk_shard_info(const gk_shard* s, int64_t* num_nodes, int64_t* lo,
                               int64_t* hi, int64_t* local_arcs, int64_t* block);
/* Kernels this shard has launched so far (telemetry for the bench line). */
GK_API int64_t gk_shard_launches(const gk_shard* s);
/* This rank's rows to host arrays (hi-lo+1 local offsets, local_arcs ids; either may be NULL). */
GK_API gk_status gk_shard_download(const gk_shard* s, int64_t* local_offsets, uint32_t* neighbors);
/* Stream of this shard's traversals (NULL: its own). */
GK_API gk_status gk_shard_set_stream(gk_shard* s, void* cuda_stream);
GK_API gk_status gk_shard_join_local(gk_shard* const* shards, int nranks);
GK_API int64_t gk_shard_handle_size(void);
GK_API gk_status gk_shard_export(const gk_shard* s, void* handle_out);
GK_API gk_status gk_shard_connect(gk_shard* s, const void* handles);
GK_API gk_status gk_shard_gather_dead(gk_shard* s);
/* One traversal of a local group (call on rank 0).  parents_out[q] /
 * depths_out[q]: rank q's owned vertices (host arrays; the arrays of
 * pointers and their entries may be NULL).  stats: device_ms of the whole
 * trial (allocation, initialisation, kernel), the step log, and (with
 * want_counts) reached / component_edges of the whole graph. */
GK_API gk_status gk_shard_group_bfs(gk_shard* rank0, uint32_t source, int64_t alpha,
                                    int64_t beta, int32_t strategy,
                                    int32_t* const* parents_out,
                                    int32_t* const* depths_out, gk_bfs_stats* stats);
/* One traversal, multi-device (collective: every rank, same arguments).
 * parent_out / depth_out: this rank's owned vertices.  With want_counts,
 * stats->reached counts this rank's reached vertices and
 * stats->component_edges their out-arcs (sum over ranks, halve).
 * *bytes_in (may be NULL) = exchange bytes this rank received. */
GK_API gk_status gk_shard_bfs(gk_shard* s, uint32_t source, int64_t alpha, int64_t beta,
                              int32_t strategy, int32_t* parent_out, int32_t* depth_out,
                              gk_bfs_stats* stats, int64_t* bytes_in);
/* Phase trace of the last traversal on this shard (rank 0 of a local
 * group): as gk_bfs_trace. */
GK_API gk_status gk_shard_trace(const gk_shard* s, uint64_t* ts_ns, char* tags, int32_t cap, int32_t* count);
/* Exchange bytes rank `rank` received in a traversal with this step log
 * (the all-gather of next per step, the claims reduce per top-down step). */
GK_API gk_status gk_shard_bytes_in(const gk_shard* s, int32_t rank, const gk_step* steps,
                                   int32_t num_steps, int64_t* out);

/* Pinned host buffers for end-to-end transfers. */
GK_API void* gk_host_alloc(int64_t bytes);
GK_API void gk_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* GK_BFS_H_ */
