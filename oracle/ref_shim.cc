// ref_shim.cc -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see gk_oracle.h).  Compiled by oracle/Makefile
// against /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libgapref.so.  Used to pin the C restatement (gk_oracle.c) and
// the CUDA path to the reference, to generate tests/golden/, and as the CPU
// baseline (bench.py cpu_baseline / --impl reference, kind "reference").
//
// Entry points wrap: GenerateKronecker/GenerateUniform (generator.hpp:56-112),
// BuildCsr (builder.hpp:54-186), the public CsrGraph constructor
// (graph.hpp:30-45), PickSources (source_picker.hpp:47-54), Bfs
// (kernels/bfs.hpp:117-177), detail::BfsDepths / VerifyBfs
// (verify.hpp:42-98), and the RunBenchmark BFS timing rule
// (benchmark.hpp:178-185: steady_clock around the Bfs call).

#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "gapkit/gapkit.hpp"
#include "ref_graph.hpp"

using namespace gapkit;
using gkref::RefGraph;

namespace {

void SetErr(char* err, int len, const std::string& s) {
  if (err && len > 0) {
    std::strncpy(err, s.c_str(), static_cast<size_t>(len - 1));
    err[len - 1] = 0;
  }
}

}  // namespace

extern "C" {

int gkr_max_threads() { return omp_get_max_threads(); }
void gkr_set_threads(int t) {
  if (t > 0) omp_set_num_threads(t);
}

// GenerateKronecker / GenerateUniform: fill 2*m interleaved uint32.
int64_t gkr_gen(int kind, int scale, int degree, uint64_t seed, uint32_t* edges) {
  GenSpec spec{kind == 0 ? GenKind::kKronecker : GenKind::kUniformRandom, scale,
               degree, seed};
  EdgeList el = kind == 0 ? GenerateKronecker(spec) : GenerateUniform(spec);
  for (size_t i = 0; i < el.edges.size(); i++) {
    edges[2 * i] = el.edges[i].src;
    edges[2 * i + 1] = el.edges[i].dst;
  }
  return static_cast<int64_t>(el.edges.size());
}

// BuildCsr(el, directed, symmetrize) over an interleaved edge array.
void* gkr_build(int64_t n, const uint32_t* edges, int64_t m, int directed,
                int symmetrize, char* err, int errlen) {
  try {
    EdgeList el;
    el.node_count = n;
    el.edges.resize(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; i++) el.edges[i] = {edges[2 * i], edges[2 * i + 1]};
    auto* h = new RefGraph;
    h->g = BuildCsr(el, directed != 0, symmetrize != 0);
    h->directed = h->g.directed();
    h->n = h->g.num_nodes();
    h->sealed = true;
    return h;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return nullptr;
  }
}

// Allocate arrays for a graph whose CSR is filled by the caller (e.g. from
// the device builder), then wrap them with the public constructor.
void* gkr_graph_alloc(int64_t n, int64_t m, int directed, int64_t** off,
                      uint32_t** nb, int64_t** in_off, uint32_t** in_nb) {
  auto* h = new RefGraph;
  h->directed = directed != 0;
  h->n = n;
  h->off.assign(static_cast<size_t>(n + 1), 0);
  h->nb.resize(static_cast<size_t>(m));
  *off = h->off.data();
  *nb = h->nb.data();
  if (h->directed) {
    h->in_off.assign(static_cast<size_t>(n + 1), 0);
    h->in_nb.resize(static_cast<size_t>(m));
    *in_off = h->in_off.data();
    *in_nb = h->in_nb.data();
  } else {
    if (in_off) *in_off = nullptr;
    if (in_nb) *in_nb = nullptr;
  }
  return h;
}

// graph.hpp:30-45 public constructor; check=1 also runs CheckInvariants.
int gkr_graph_seal(void* hp, int check, char* err, int errlen) {
  auto* h = static_cast<RefGraph*>(hp);
  h->g = CsrGraph(h->directed, false, h->n, std::move(h->off), std::move(h->nb), {},
                  std::move(h->in_off), std::move(h->in_nb));
  h->sealed = true;
  if (check) {
    if (auto msg = h->g.CheckInvariants()) {
      SetErr(err, errlen, *msg);
      return 0;
    }
  }
  return 1;
}

void gkr_graph_free(void* hp) { delete static_cast<RefGraph*>(hp); }

int64_t gkr_graph_n(void* hp) { return static_cast<RefGraph*>(hp)->g.num_nodes(); }
int64_t gkr_graph_m(void* hp) { return static_cast<RefGraph*>(hp)->g.num_edges(); }
int gkr_graph_directed(void* hp) { return static_cast<RefGraph*>(hp)->g.directed(); }

// Copy out the (sealed) CSR arrays; any pointer may be null.
void gkr_graph_arrays(void* hp, int64_t* off, uint32_t* nb, int64_t* in_off,
                      uint32_t* in_nb) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  if (off) std::memcpy(off, g.out_offsets().data(), g.out_offsets().size() * 8);
  if (nb) std::memcpy(nb, g.out_neighbors().data(), g.out_neighbors().size() * 4);
  if (in_off) std::memcpy(in_off, g.in_offsets().data(), g.in_offsets().size() * 8);
  if (in_nb) std::memcpy(in_nb, g.in_neighbors().data(), g.in_neighbors().size() * 4);
}

int gkr_pick_sources(void* hp, int64_t count, uint64_t seed, uint32_t* out,
                     char* err, int errlen) {
  try {
    std::vector<NodeId> s = PickSources(static_cast<RefGraph*>(hp)->g, count, seed);
    std::memcpy(out, s.data(), s.size() * 4);
    return 1;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 0;
  }
}

// Bfs(g, src, {alpha, beta, strategy}); 0 + message on ConfigError.
int gkr_bfs(void* hp, uint32_t src, int64_t alpha, int64_t beta, int strategy,
            int32_t* parent, char* err, int errlen) {
  try {
    BfsOptions o;
    o.alpha = alpha;
    o.beta = beta;
    o.strategy = static_cast<BfsStrategy>(strategy);
    ParentArray p = Bfs(static_cast<RefGraph*>(hp)->g, src, o);
    std::memcpy(parent, p.data(), p.size() * 4);
    return 1;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 0;
  }
}

// RunBenchmark's BFS case (benchmark.hpp:181-185): steady_clock around one
// Bfs call (allocation included); returns seconds per source in secs[],
// and the parent digest of each trial in digests[] (may be null).
void gkr_bfs_timed(void* hp, const uint32_t* sources, int count, int64_t alpha,
                   int64_t beta, double* secs, uint64_t* digests) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  for (int i = 0; i < count; i++) {
    Timer t;
    t.Start();
    ParentArray p = Bfs(g, sources[i], {.alpha = alpha, .beta = beta});
    t.Stop();
    secs[i] = t.Seconds();
    if (digests) digests[i] = HashBytes(p.data(), p.size() * sizeof(ParentEntry));
  }
}

// Schedule replay driven by the reference's own step functions
// (detail::BfsTopDownStep / BfsBottomUpStep / QueueToBitmap / BitmapToQueue,
// bfs.hpp:47-113) under the driver loop of bfs.hpp:125-169, restated here
// only to record each step's direction and counters.  Returns the number of
// steps (records at most max_steps); parent gets the final ParentArray.
int64_t gkr_bfs_schedule(void* hp, uint32_t src, int64_t alpha, int64_t beta, int strategy,
                         int32_t* dirs, int64_t* frontier, int64_t* result, int64_t* etc_out,
                         int64_t max_steps, int32_t* parent_out) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  const int64_t n = g.num_nodes();
  const bool encode = strategy != static_cast<int>(BfsStrategy::kTopDownRescan);
  ParentArray parent(n);
  for (int64_t v = 0; v < n; v++) {
    int64_t degree = encode ? g.out_degree(static_cast<NodeId>(v)) : 0;
    parent[v] = degree != 0 ? static_cast<ParentEntry>(-degree) : -1;
  }
  parent[src] = static_cast<ParentEntry>(src);
  SlidingQueue<NodeId> queue(n);
  queue.PushBack(src);
  queue.SlideWindow();
  Bitmap front(n), next(n);
  int64_t edges_to_check = g.num_edges();
  int64_t scout_count = g.out_degree(src);
  int64_t ns = 0;
  auto rec = [&](int d, int64_t f, int64_t r) {
    if (ns < max_steps) {
      dirs[ns] = d;
      frontier[ns] = f;
      result[ns] = r;
      etc_out[ns] = edges_to_check;
    }
    ns++;
  };
  while (!queue.Empty()) {
    if (strategy == 0 && scout_count > edges_to_check / alpha) {
      detail::QueueToBitmap(queue, front);
      int64_t awake_count = queue.Size();
      queue.SlideWindow();
      int64_t old_awake_count;
      do {
        old_awake_count = awake_count;
        awake_count = detail::BfsBottomUpStep(g, parent, front, next);
        front.Swap(next);
        rec('B', old_awake_count, awake_count);
      } while (awake_count >= old_awake_count || awake_count > n / beta);
      detail::BitmapToQueue(g, front, queue);
      scout_count = 1;
    } else {
      edges_to_check -= scout_count;
      int64_t fsize = static_cast<int64_t>(queue.Size());
      scout_count = detail::BfsTopDownStep(g, parent, queue);
      queue.SlideWindow();
      if (strategy == 2) {
        int64_t tot = 0;
        for (auto it = queue.begin(); it < queue.end(); ++it) tot += g.out_degree(*it);
        scout_count = tot;
      }
      rec('T', fsize, scout_count);
    }
  }
  for (int64_t v = 0; v < n; v++)
    if (parent[v] < 0) parent[v] = -1;
  if (parent_out) std::memcpy(parent_out, parent.data(), parent.size() * 4);
  return ns;
}

// WriteSerialized / ReadSerialized (io.hpp:364-456) for the .sg fixtures.
int gkr_write_sg(void* hp, const char* path, int weighted_seed_or_minus1, char* err, int errlen) {
  try {
    const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
    if (weighted_seed_or_minus1 >= 0)
      WriteSerialized(EnsureWeighted(g, static_cast<uint64_t>(weighted_seed_or_minus1)), path);
    else
      WriteSerialized(g, path);
    return 1;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 0;
  }
}

void* gkr_read_sg(const char* path, char* err, int errlen) {
  try {
    auto* h = new RefGraph;
    h->g = ReadSerialized(path);
    h->directed = h->g.directed();
    h->n = h->g.num_nodes();
    h->sealed = true;
    return h;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return nullptr;
  }
}

void gkr_bfs_depths(void* hp, uint32_t src, int32_t* depth) {
  std::vector<int32_t> d = detail::BfsDepths(static_cast<RefGraph*>(hp)->g, src);
  std::memcpy(depth, d.data(), d.size() * 4);
}

int gkr_verify_bfs(void* hp, uint32_t src, const int32_t* parent, char* msg,
                   int msglen) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  ParentArray p(parent, parent + g.num_nodes());
  VerifyReport r = VerifyBfs(g, src, p);
  SetErr(msg, msglen, r.failure_detail);
  return r.ok ? 1 : 0;
}

// Brandes (kernels/betweenness.hpp:84-145).  Returns 0, or 1 with the
// ConfigError message in err.
int gkr_brandes(void* hp, const uint32_t* sources, int64_t count, float* scores, char* err,
                int errlen) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  std::vector<NodeId> s(sources, sources + count);
  try {
    ScoreArray sc = Brandes(g, s);
    std::memcpy(scores, sc.data(), sc.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 1;
  }
}

// VerifyBetweenness (verify.hpp:216-270), default tolerance 1e-4.
int gkr_verify_bc(void* hp, const uint32_t* sources, int64_t count, const float* scores, char* msg,
                  int msglen) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  std::vector<NodeId> s(sources, sources + count);
  ScoreArray sc(scores, scores + g.num_nodes());
  VerifyReport r = VerifyBetweenness(g, s, sc);
  SetErr(msg, msglen, r.failure_detail);
  return r.ok ? 1 : 0;
}

}  // extern "C"
