// integration_snippet.cc -- INTEGRATION.md §2's snippet, verbatim, as a
// program: the reference's own graph and harness calls with the B200 BFS
// dropped in through gapkit_b200/ref_binding.hpp.  Compiled (and linked)
// by paper_1508_03619_b200/host/Makefile; tests/test_host_cpp.py checks it
// builds, and runs it where a GPU exists.
#include <cstdio>

#include "gapkit/gapkit.hpp"            // the reference, unmodified
#include "gapkit_b200/ref_binding.hpp"  // gapkit::b200::Bfs over include/gk_bfs.h

int main() {
  using namespace gapkit;
  CsrGraph g = BuildCsr(GenerateKronecker({GenKind::kKronecker, 16, 16, kDefaultSeed}), false, true);
  for (NodeId s : PickSources(g, 8)) {
    ParentArray p = b200::Bfs(g, s, {.alpha = 15, .beta = 18});
    if (!VerifyBfs(g, s, p).ok) return 1;
  }
  std::printf("ok\n");
  return 0;
}
