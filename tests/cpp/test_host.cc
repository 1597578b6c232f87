// Driver for the C++ host-surface tests (tests/test_host_cpp.py runs it).
//   test_host hash (kron|urand|kronp) SCALE SEED  -> FNV of edges / offsets / neighbours (host build)
//   test_host grid ROWS COLS SEED                  -> same for the road-like grid
//   test_host pick (kron|urand) SCALE SEED COUNT   -> PickSources
//   test_host errors                               -> ConfigError paths that need no device
//   test_host gpu                                  -> Bfs through libgk_bfs.so (needs a GPU)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gapkit_b200/betweenness.hpp"
#include "gapkit_b200/bfs.hpp"
#include "gapkit_b200/builder.hpp"
#include "gapkit_b200/generator.hpp"
#include "gapkit_b200/harness.hpp"

using namespace gapkit;

#define CHECK(c)                                                           \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

template <typename F>
static bool Throws(F f, const char* needle) {
  try {
    f();
  } catch (const ConfigError& e) {
    return std::strstr(e.what(), needle) != nullptr;
  } catch (...) {
    return false;
  }
  return false;
}

static CsrGraph Build(const std::string& kind, int scale, uint64_t seed, EdgeList* keep = nullptr) {
  GenSpec spec{kind == "urand" ? GenKind::kUniformRandom : GenKind::kKronecker, scale, 16, seed};
  EdgeList el = kind == "urand" ? GenerateUniform(spec) : GenerateKronecker(spec);
  if (kind == "kronp") PermuteIds(el, scale, seed);
  if (keep) *keep = el;
  return BuildCsr(el, false, true);
}

static void PrintHashes(const EdgeList& el, const CsrGraph& g) {
  std::vector<uint32_t> flat;
  flat.reserve(2 * el.edges.size());
  for (const Edge& e : el.edges) {
    flat.push_back(e.src);
    flat.push_back(e.dst);
  }
  std::printf("%lld %lld %016llx %016llx %016llx\n", (long long)g.num_nodes(), (long long)g.num_edges(),
              (unsigned long long)HashBytes(flat.data(), flat.size() * 4),
              (unsigned long long)HashBytes(g.out_offsets().data(), g.out_offsets().size() * 8),
              (unsigned long long)HashBytes(g.out_neighbors().data(), g.out_neighbors().size() * 4));
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string cmd = argv[1];
  if (cmd == "hash") {
    EdgeList el;
    CsrGraph g = Build(argv[2], std::atoi(argv[3]), std::strtoull(argv[4], nullptr, 10), &el);
    PrintHashes(el, g);
    return 0;
  }
  if (cmd == "grid") {
    EdgeList el = GenerateGrid(std::atoll(argv[2]), std::atoll(argv[3]), 0.15, 0.02, std::strtoull(argv[4], nullptr, 10));
    PrintHashes(el, BuildCsr(el, false, true));
    return 0;
  }
  if (cmd == "pick") {
    CsrGraph g = Build(argv[2], std::atoi(argv[3]), std::strtoull(argv[4], nullptr, 10));
    for (NodeId s : PickSources(g, std::atoll(argv[5]), std::strtoull(argv[4], nullptr, 10))) std::printf("%u ", s);
    std::printf("\n");
    return 0;
  }
  if (cmd == "errors") {
    EdgeList el;
    el.Add(0, 1);
    el.Add(1, 2);
    CsrGraph path = BuildCsr(el, false, true);
    CHECK(Throws([&] { Bfs(path, 17); }, "bfs source out of range"));
    CHECK(Throws([&] { Bfs(path, 0, {.alpha = 0}); }, "bfs alpha and beta must be positive"));
    EdgeList empty;
    empty.node_count = 4;
    CsrGraph e = BuildCsr(empty, false, true);
    CHECK(Throws([&] { PickSources(e, 1); }, "no edges"));
    CHECK(Throws([&] { GenerateKronecker({GenKind::kKronecker, 40}); }, "scale"));
    // builder: self-loops and duplicates dropped, lists sorted (test_builder.cc:14-31)
    EdgeList d;
    d.Add(2, 0);
    d.Add(0, 2);
    d.Add(1, 1);
    d.Add(0, 1);
    d.Add(0, 1);
    CsrGraph b = BuildCsr(d, true, false);
    CHECK(b.num_edges() == 3 && b.out_neighbors() == (std::vector<NodeId>{1, 2, 0}));
    CHECK(b.in_neighbors() == (std::vector<NodeId>{2, 0, 0}));
    CHECK(!b.CheckInvariants().has_value());
    // verifier tampers (test_verify.cc:13-57)
    ParentArray good = {0, 0, 1};
    CHECK(VerifyBfs(path, 0, good).ok);
    ParentArray bad = good;
    bad[2] = 0;
    CHECK(!VerifyBfs(path, 0, bad).ok && VerifyBfs(path, 0, bad).failure_detail.find("no edge") != std::string::npos);
    bad = good;
    bad[2] = -1;
    CHECK(VerifyBfs(path, 0, bad).failure_detail.find("unreached") != std::string::npos);
    // host betweenness checker, known answers (no device pass involved):
    // path 0-1-2 from every source -> only the middle vertex scores;
    // diamond 0-{1,2}-3 from 0 -> 1 and 2 each carry half of 0->3
    std::vector<NodeId> p3 = {0, 1, 2};
    CHECK(VerifyBetweenness(path, p3, ScoreArray{0.0f, 1.0f, 0.0f}).ok);
    CHECK(VerifyBetweenness(path, p3, ScoreArray{0.0f, 0.5f, 0.0f}).failure_detail.find("vertex 1") !=
          std::string::npos);
    CHECK(!VerifyBetweenness(path, p3, ScoreArray{0.0f, 1.0f}).ok);
    EdgeList dm;
    dm.Add(0, 1);
    dm.Add(0, 2);
    dm.Add(1, 3);
    dm.Add(2, 3);
    dm.Add(3, 4);
    CsrGraph diamond = BuildCsr(dm, false, true);
    std::vector<NodeId> s0 = {0};
    // from 0: delta(3) = 1 (vertex 4), delta(1) = delta(2) = (1 + 1) / 2 = 1
    CHECK(VerifyBetweenness(diamond, s0, ScoreArray{0.0f, 1.0f, 1.0f, 1.0f, 0.0f}).ok);
    std::vector<NodeId> s4 = {4};
    // from 4: delta(3) = 3, delta(1) = delta(2) = 1/2 -> normalised 1/6
    CHECK(VerifyBetweenness(diamond, s4, ScoreArray{0.0f, 1.0f / 6, 1.0f / 6, 1.0f, 0.0f}).ok);
    std::printf("errors ok\n");
    return 0;
  }
  if (cmd == "bc") {  // test_kernels_source.cc:136-158 through the device
    EdgeList star;
    star.node_count = 5;
    for (NodeId v = 0; v < 4; v++) star.Add(4, v);
    CsrGraph sg = BuildCsr(star, false, true);
    std::vector<NodeId> all = {0, 1, 2, 3, 4};
    ScoreArray sc = Brandes(sg, all);
    CHECK(sc[4] == 1.0f);
    for (int leaf = 0; leaf < 4; leaf++) CHECK(sc[leaf] == 0.0f);
    EdgeList p2;
    p2.Add(0, 1);
    std::vector<NodeId> zero = {0};
    ScoreArray pz = Brandes(BuildCsr(p2, false, true), zero);
    CHECK(pz[0] == 0.0f && pz[1] == 0.0f);
    EdgeList e3;
    e3.node_count = 3;
    e3.Add(0, 1);
    CsrGraph g3 = BuildCsr(e3, false, true);
    std::vector<NodeId> none, iso = {2};
    CHECK(Throws([&] { Brandes(g3, none); }, "betweenness requires at least one source"));
    CHECK(Throws([&] { Brandes(g3, iso); }, "zero out-degree"));
    CsrGraph k = Build("kron", 10, kDefaultSeed);
    std::vector<NodeId> src = PickSources(k, 4);
    ScoreArray ks = Brandes(k, src);
    for (Score x : ks) CHECK(x >= 0.0f && x <= 1.0f);
    std::printf("bc ok\n");
    return 0;
  }
  if (cmd == "gpu") {
    EdgeList el;
    el.Add(0, 1);
    el.Add(1, 2);
    CsrGraph path = BuildCsr(el, false, true);
    CHECK(Bfs(path, 0) == (ParentArray{0, 0, 1}));  // test_kernels_source.cc:13-17
    EdgeList el4;
    el4.node_count = 4;
    el4.Add(0, 1);
    el4.Add(1, 2);
    CHECK(Bfs(BuildCsr(el4, false, true), 0)[3] == -1);  // :19-23
    CHECK(Throws([&] { Bfs(path, 17); }, "bfs source out of range"));
    for (const char* kind : {"kron", "urand", "kronp"}) {  // :31-40
      CsrGraph g = Build(kind, 12, kDefaultSeed);
      for (NodeId s : PickSources(g, 16)) {
        for (BfsStrategy st : {BfsStrategy::kDirectionOptimizing, BfsStrategy::kTopDownOnly,
                               BfsStrategy::kTopDownRescan}) {
          VerifyReport r = VerifyBfs(g, s, Bfs(g, s, {.strategy = st}));
          if (!r.ok) std::fprintf(stderr, "%s %u: %s\n", kind, s, r.failure_detail.c_str());
          CHECK(r.ok);
        }
      }
    }
    // device-built graph equals the host build (generator + BuildCsr)
    CsrGraph hg = Build("kronp", 14, 99);
    CsrGraph dg = GenerateOnDevice({GenKind::kKronecker, 14, 16, 99}, true);
    dg.EnsureHostArrays();
    CHECK(hg.out_offsets() == dg.out_offsets() && hg.out_neighbors() == dg.out_neighbors());
    CHECK(PickSources(hg, 8, 5) == PickSources(dg, 8, 5));
    // directed graph, bottom-up on in-edges (:55-67)
    EdgeList del = GenerateKronecker({GenKind::kKronecker, 11, 16, 11});
    CsrGraph dirg = BuildCsr(del, true, false);
    for (NodeId s : PickSources(dirg, 8)) CHECK(VerifyBfs(dirg, s, Bfs(dirg, s, {.alpha = 1, .beta = 1})).ok);
    // harness
    BenchPlan plan;
    plan.trials = 8;
    BenchReport rep = RunBenchmark(hg, plan, true, "kronp14");
    CHECK(rep.trials.size() == 8 && rep.AllVerified() && rep.HmeanDeviceGteps() > 0);
    std::printf("gpu ok\n");
    return 0;
  }
  return 2;
}
