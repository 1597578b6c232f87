// cpp_e2e.cc -- where gapkit::Bfs(g, src)'s host wall clock goes (kron S):
// FreshVector alone, Bfs with and without telemetry, gk_bfs into pinned.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "gapkit_b200/bfs.hpp"
#include "gapkit_b200/generator.hpp"
#include "gapkit_b200/harness.hpp"

using namespace gapkit;
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 27;
  CsrGraph g = GenerateOnDevice({GenKind::kKronecker, scale, 16, kDefaultSeed}, true);
  std::vector<NodeId> src = PickSources(g, 6);
  const size_t n = g.num_nodes();
  int32_t* pin = static_cast<int32_t*>(gk_host_alloc(4 * n));
  for (int i = 0; i < 6; i++) {
    double t0 = now();
    { auto v = gk_host::FreshVector<int32_t>(n); }
    double t1 = now();
    { ParentArray p = Bfs(g, src[i]); }
    double t2 = now();
    BfsTelemetry tel;
    { ParentArray p = Bfs(g, src[i], {}, &tel); }
    double t3 = now();
    gk_bfs(g.device(), src[i], 15, 18, 0, pin, nullptr, nullptr);
    double t4 = now();
    gk_bfs(g.device(), src[i], 15, 18, 0, nullptr, nullptr, nullptr);
    double t5 = now();
    std::vector<int32_t> plain(n);
    double t6 = now();
    gk_bfs(g.device(), src[i], 15, 18, 0, plain.data(), nullptr, nullptr);
    double t7 = now();
    printf("src %u: FreshVector %.1f ms | Bfs %.1f | Bfs+telemetry %.1f | gk_bfs->pinned %.1f | gk_bfs no copy %.1f"
           " | vector(n) %.1f | gk_bfs->faulted pageable %.1f\n",
           src[i], (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3,
           (t6 - t5) * 1e3, (t7 - t6) * 1e3);
  }
  gk_host_free(pin);
  return 0;
}
