// ref_bench.cc -- the reference arm's graphs and trials for bench.py
// --impl reference and the full-size parity tests.
//
// TEST / BASELINE INFRASTRUCTURE ONLY (see gk_oracle.h).  Compiled into
// oracle/_ref/libgapref.so next to ref_shim.cc against the UNMODIFIED
// reference headers (oracle/Makefile).  Nothing here touches libgk_bfs.so:
// the reference arm builds its own graph on the host and times the
// reference's own Bfs on it.
//
// A bench configuration's graph, built the way the device builds it:
//   1. the reference's GenerateKronecker / GenerateUniform
//      (generator.hpp:56-112), unmodified, or the road-like grid (a new
//      generator: gk_oracle.c's restatement, the same as the device's);
//   2. the seeded vertex-ID bijection applied to every endpoint (new;
//      gk_oracle.c gko_permute, the same as the device's);
//   3. BuildCsr(el, false, true) semantics (builder.hpp:54-186: mirror every
//      edge, drop self-loops, sort each list, drop duplicates) by a 64-bit
//      OpenMP builder -- the reference's own BuildCsr stops at 2^32 arcs
//      ("edge list too large for the builder", builder.hpp:71-73), which
//      every scale-27 configuration exceeds.  tests/test_oracle.py checks
//      it byte-identical to BuildCsr where the reference builder can run;
//   4. the public CsrGraph constructor (graph.hpp:30-45).
// Trials follow RunBenchmark's BFS case (benchmark.hpp:178-185): steady_clock
// around one Bfs call, allocation of the result included.

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "gapkit/gapkit.hpp"
#include "gk_oracle.h"
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

// Exclusive prefix sum of a[0..n) into a (a[n] receives the total), in
// parallel: per-thread block sums, then a pass adding the block offsets.
void ParallelScan(int64_t* a, int64_t n) {
  const int nt = omp_get_max_threads();
  std::vector<int64_t> part(static_cast<size_t>(nt) + 1, 0);
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    int64_t s = 0;
    for (int64_t i = lo; i < hi; i++) s += a[i];
    part[t + 1] = s;
#pragma omp barrier
#pragma omp single
    for (int i = 0; i < nt; i++) part[i + 1] += part[i];
    int64_t run = part[t];
    for (int64_t i = lo; i < hi; i++) {
      const int64_t x = a[i];
      a[i] = run;
      run += x;
    }
  }
  a[n] = part[nt];
}

// BuildCsr(el, directed=false, symmetrize=true) for any edge count, as a
// two-level radix build so every pass stays cache-local:
//   1. each thread counts its slice of the edge list's arcs (both
//      directions, self-loops dropped) per source bucket of 2^kBucketBits
//      vertices, and scatters them as (local source << 32 | target) into
//      the buckets (one write stream per bucket and thread);
//   2. per bucket: counting sort by source, each list sorted and
//      deduplicated (= BuildCsr's per-list sort + unique), the deduplicated
//      lists compacted into the bucket's own space, degrees recorded;
//   3. prefix sum of the degrees, then each bucket's lists copied to the
//      final neighbour array.
CsrGraph BuildSymmetric64(EdgeList&& el, int64_t n) {
  constexpr int kBucketBits = 15;
  const int64_t m = static_cast<int64_t>(el.edges.size());
  const int64_t nbk = (n + (int64_t{1} << kBucketBits) - 1) >> kBucketBits;
  const int nt = omp_get_max_threads();
  std::vector<int64_t> pos(static_cast<size_t>(nt) * nbk + 1, 0);  // [bucket][thread]
  auto slice = [&](int t, int64_t& lo, int64_t& hi) {
    lo = m * t / nt;
    hi = m * (t + 1) / nt;
  };
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    int64_t lo, hi;
    slice(t, lo, hi);
    std::vector<int64_t> h(static_cast<size_t>(nbk), 0);
    for (int64_t i = lo; i < hi; i++) {
      const Edge e = el.edges[i];
      if (e.src == e.dst) continue;
      h[e.src >> kBucketBits]++;
      h[e.dst >> kBucketBits]++;
    }
    for (int64_t b = 0; b < nbk; b++) pos[b * nt + t] = h[b];
  }
  ParallelScan(pos.data(), static_cast<int64_t>(nt) * nbk);
  const int64_t raw_m = pos[static_cast<size_t>(nt) * nbk];
  std::vector<uint64_t> pairs(static_cast<size_t>(raw_m));
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    int64_t lo, hi;
    slice(t, lo, hi);
    std::vector<int64_t> cur(static_cast<size_t>(nbk));
    for (int64_t b = 0; b < nbk; b++) cur[b] = pos[b * nt + t];
    constexpr uint32_t kMask = (1u << kBucketBits) - 1;
    for (int64_t i = lo; i < hi; i++) {
      const Edge e = el.edges[i];
      if (e.src == e.dst) continue;
      pairs[cur[e.src >> kBucketBits]++] = (uint64_t{e.src & kMask} << 32) | e.dst;
      pairs[cur[e.dst >> kBucketBits]++] = (uint64_t{e.dst & kMask} << 32) | e.src;
    }
  }
  el.edges.clear();
  el.edges.shrink_to_fit();
  std::vector<int64_t> out_off(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel
  {
    std::vector<uint32_t> tmp;
    std::vector<int64_t> cnt;
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < nbk; b++) {
      const int64_t v0 = b << kBucketBits;
      const int64_t nv = std::min<int64_t>(int64_t{1} << kBucketBits, n - v0);
      const int64_t lo = pos[b * nt], hi = pos[(b + 1) * nt];
      cnt.assign(static_cast<size_t>(nv) + 1, 0);
      for (int64_t i = lo; i < hi; i++) cnt[(pairs[i] >> 32) + 1]++;
      for (int64_t v = 0; v < nv; v++) cnt[v + 1] += cnt[v];
      tmp.resize(static_cast<size_t>(hi - lo));
      {
        std::vector<int64_t> c(cnt.begin(), cnt.end() - 1);
        for (int64_t i = lo; i < hi; i++) tmp[c[pairs[i] >> 32]++] = static_cast<uint32_t>(pairs[i]);
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(pairs.data() + lo);  // compacted lists, in place
      int64_t w = 0;
      for (int64_t v = 0; v < nv; v++) {
        uint32_t* a = tmp.data() + cnt[v];
        uint32_t* z = tmp.data() + cnt[v + 1];
        std::sort(a, z);
        z = std::unique(a, z);
        out_off[v0 + v] = z - a;
        std::memcpy(dst + w, a, sizeof(uint32_t) * (z - a));
        w += z - a;
      }
    }
  }
  ParallelScan(out_off.data(), n);
  std::vector<NodeId> nb(static_cast<size_t>(out_off[n]));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t b = 0; b < nbk; b++) {
    const int64_t v0 = b << kBucketBits;
    const int64_t v1 = std::min<int64_t>(v0 + (int64_t{1} << kBucketBits), n);
    std::memcpy(nb.data() + out_off[v0], pairs.data() + pos[b * nt], sizeof(NodeId) * (out_off[v1] - out_off[v0]));
  }
  pairs.clear();
  pairs.shrink_to_fit();
  return CsrGraph(false, false, n, std::move(out_off), std::move(nb), {});
}

}  // namespace

extern "C" {

// kind 0 Kronecker, 1 uniform, 2 grid (rows, cols in scale/degree slots:
// rows = scale, cols = degree, p_delete / p_diag).  Returns a handle usable
// with every gkr_* entry point of ref_shim.cc, or null with the message.
void* gkr_bench_graph(int kind, int64_t scale_or_rows, int64_t degree_or_cols, uint64_t seed, int permute,
                      double p_delete, double p_diag, char* err, int errlen) {
  try {
    EdgeList el;
    int64_t n = 0;
    if (kind == 0 || kind == 1) {
      const int scale = static_cast<int>(scale_or_rows);
      GenSpec spec{kind == 0 ? GenKind::kKronecker : GenKind::kUniformRandom, scale,
                   static_cast<int>(degree_or_cols), seed};
      el = kind == 0 ? GenerateKronecker(spec) : GenerateUniform(spec);
      n = int64_t{1} << scale;
      if (permute) {
        uint64_t keys[8];
        gko_perm_keys(seed, scale, keys);
        const int64_t m = static_cast<int64_t>(el.edges.size());
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; i++) {
          el.edges[i].src = gko_permute(el.edges[i].src, scale, keys);
          el.edges[i].dst = gko_permute(el.edges[i].dst, scale, keys);
        }
      }
    } else if (kind == 2) {
      const int64_t rows = scale_or_rows, cols = degree_or_cols;
      std::vector<uint32_t> e(2 * static_cast<size_t>(gko_grid_max_edges(rows, cols)));
      const int64_t m = gko_gen_grid(rows, cols, p_delete, p_diag, seed, e.data());
      el.edges.resize(static_cast<size_t>(m));
      for (int64_t i = 0; i < m; i++) el.edges[i] = {e[2 * i], e[2 * i + 1]};
      n = rows * cols;
    } else {
      SetErr(err, errlen, "unknown graph kind");
      return nullptr;
    }
    auto* h = new RefGraph;
    h->g = BuildSymmetric64(std::move(el), n);
    h->n = n;
    h->sealed = true;
    return h;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return nullptr;
  }
}

// BuildCsr-equivalence check hook: the 64-bit builder on a caller edge list.
void* gkr_build64(int64_t n, const uint32_t* edges, int64_t m) {
  EdgeList el;
  el.edges.resize(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; i++) el.edges[i] = {edges[2 * i], edges[2 * i + 1]};
  auto* h = new RefGraph;
  h->g = BuildSymmetric64(std::move(el), n);
  h->n = n;
  h->sealed = true;
  return h;
}

// Read-only views of a sealed graph's out-CSR (no copy).
void gkr_graph_views(void* hp, const int64_t** off, const uint32_t** nb) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  *off = g.out_offsets().data();
  *nb = g.out_neighbors().data();
}

// Undirected edges in the component a ParentArray reached: (sum of
// out-degree over v with parent >= 0) / (directed ? 1 : 2).
int64_t gkr_component_edges(void* hp, const int32_t* parent) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  const int64_t n = g.num_nodes();
  const int64_t* off = g.out_offsets().data();
  int64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t v = 0; v < n; v++)
    if (parent[v] >= 0) s += off[v + 1] - off[v];
  return g.directed() ? s : s / 2;
}

// RunBenchmark's BFS trial loop (benchmark.hpp:178-185) over count sources:
// secs[i] = steady_clock seconds of Bfs(g, sources[i]) (allocation of the
// ParentArray included); mcc[i] = component edges of that result (untimed).
void gkr_bfs_trials(void* hp, const uint32_t* sources, int count, int64_t alpha, int64_t beta, double* secs,
                    int64_t* mcc) {
  const CsrGraph& g = static_cast<RefGraph*>(hp)->g;
  for (int i = 0; i < count; i++) {
    Timer t;
    t.Start();
    ParentArray p = Bfs(g, sources[i], {.alpha = alpha, .beta = beta});
    t.Stop();
    secs[i] = t.Seconds();
    if (mcc) mcc[i] = gkr_component_edges(hp, p.data());
  }
}

}  // extern "C"
