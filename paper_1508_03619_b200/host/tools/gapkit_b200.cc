// gapkit_b200 -- benchmark CLI on the B200 (the reference's `gapkit bfs` and
// `gapkit bc` subcommands, tools/gapkit.cc:47-152, 232-260, with a
// hand-rolled parser because CLI11 is not vendored).
//
//   gapkit_b200 bfs|bc (-f FILE.sg | -g SCALE | -u SCALE | --grid RxC) [-k DEGREE] [-n TRIALS]
//               [-r SOURCE] [-i SOURCES_PER_TRIAL] [-v] [-s] [--seed S] [--no-permute] [--host-build]
//               [--threads T] [--no-model] [--peak-gbs GB/s] [-o FILE.csv]
//
// -s/--symmetrize treats a file's graph as undirected (gapkit.cc:57-58;
// LoadGraph, io.hpp:461-468: a directed .sg is flattened and rebuilt
// symmetrized).  The CSV adds m_cc, the B_sec byte model, its roofline
// fraction against --peak-gbs and the GPU count to the reference's columns
// (--no-model skips the untimed model pass).
//
// bc follows the reference's plan (benchmark.hpp:75): 16 trials x 4 sources
// by default, -i sets the sources per trial.
//
// -g/-u generate a Kronecker / uniform graph (generator.hpp:56-112) and build
// it symmetrized (gapkit.cc:89-96); Kronecker IDs are permuted (BASELINE
// configs 1/3/5) unless --no-permute.  By default generation and the CSR
// build run on the device (bit-identical to the host path, which
// --host-build selects).  Trials follow the reference harness: one picker
// sequence, one timed Bfs per trial, untimed verification with -v.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>

#include "gapkit_b200/betweenness.hpp"
#include "gapkit_b200/bfs.hpp"
#include "gapkit_b200/builder.hpp"
#include "gapkit_b200/generator.hpp"
#include "gapkit_b200/harness.hpp"
#include "gapkit_b200/io.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

int Usage(const char* argv0) {
  std::fprintf(stderr,
               "usage: %s bfs|bc (-f FILE.sg | -g SCALE | -u SCALE | --grid RxC) [-k DEGREE] [-n TRIALS]\n"
               "          [-r SOURCE] [-i SOURCES_PER_TRIAL] [-v] [-s] [--seed S] [--no-permute] [--host-build]\n"
               "          [--threads T] [--no-model] [--peak-gbs GB/s] [-o FILE.csv]\n",
               argv0);
  return 2;
}

bool ParseInt(const char* s, long long* out) {
  char* end = nullptr;
  *out = std::strtoll(s, &end, 10);
  return end && *end == 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || (std::strcmp(argv[1], "bfs") != 0 && std::strcmp(argv[1], "bc") != 0)) return Usage(argv[0]);
  const bool bc = std::strcmp(argv[1], "bc") == 0;
  long long kron = -1, urand = -1, degree = 16, trials = bc ? 16 : 64, fixed = -1, threads = 0, per_trial = 4;
  long long rows = 0, cols = 0;
  unsigned long long seed = gapkit::kDefaultSeed;
  bool verify = false, permute = true, host_build = false, symmetrize = false, model = true;
  double peak_gbs = 6550.7;
  std::string output, file;
  for (int i = 2; i < argc; i++) {
    std::string a = argv[i];
    auto need = [&](long long* dst) {
      if (i + 1 >= argc || !ParseInt(argv[++i], dst)) {
        std::fprintf(stderr, "invalid or missing value for %s\n", a.c_str());
        std::exit(2);
      }
    };
    if (a == "-g" || a == "--kron") need(&kron);
    else if (a == "-u" || a == "--urand") need(&urand);
    else if (a == "-k" || a == "--degree") need(&degree);
    else if (a == "-n") need(&trials);
    else if (a == "-i") need(&per_trial);
    else if (a == "-r") need(&fixed);
    else if (a == "--threads") need(&threads);
    else if (a == "--seed") {
      long long s;
      need(&s);
      seed = static_cast<unsigned long long>(s);
    } else if (a == "-v") verify = true;
    else if (a == "-s" || a == "--symmetrize") symmetrize = true;
    else if (a == "--no-model") model = false;
    else if (a == "--peak-gbs") {
      if (i + 1 >= argc || std::sscanf(argv[++i], "%lf", &peak_gbs) != 1 || peak_gbs <= 0) return Usage(argv[0]);
    }
    else if (a == "--no-permute") permute = false;
    else if (a == "--host-build") host_build = true;
    else if (a == "-f" || a == "--file") {
      if (i + 1 >= argc) return Usage(argv[0]);
      file = argv[++i];
    } else if (a == "-o" || a == "--output") {
      if (i + 1 >= argc) return Usage(argv[0]);
      output = argv[++i];
    } else if (a == "--grid") {
      if (i + 1 >= argc || std::sscanf(argv[++i], "%lldx%lld", &rows, &cols) != 2) return Usage(argv[0]);
    } else {
      std::fprintf(stderr, "unknown option %s\n", a.c_str());
      return Usage(argv[0]);
    }
  }
  if (threads <= 0) {  // gapkit.cc:68-76
    if (const char* env = std::getenv("GAPKIT_THREADS")) threads = std::atoi(env);
  }
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(static_cast<int>(threads));
#endif
  try {
    const int sources = (kron >= 0) + (urand >= 0) + (rows > 0) + !file.empty();
    if (sources != 1) throw gapkit::ConfigError("exactly one graph source required (-f, -g, -u, or --grid)");
    gapkit::CsrGraph g;
    std::string name;
    if (!file.empty()) {  // gapkit.cc:85-88 (serialized formats; text formats are out of scope)
      const auto slash = file.find_last_of('/');
      name = file.substr(slash == std::string::npos ? 0 : slash + 1);
      name = name.substr(0, name.find_last_of('.'));
      g = gapkit::ReadSerializedOnDevice(file);
      if (symmetrize && g.directed()) {  // io.hpp:466-467: BuildCsr(FlattenToEdgeList(g), false, true)
        g.EnsureHostArrays();
        gapkit::EdgeList el;
        el.node_count = g.num_nodes();
        for (int64_t u = 0; u < g.num_nodes(); u++)
          for (gapkit::NodeId v : g.out_neigh(static_cast<gapkit::NodeId>(u)))
            el.edges.push_back({static_cast<gapkit::NodeId>(u), v});
        g = gapkit::BuildCsr(el, false, true);
      }
    } else if (rows > 0) {
      name = "grid" + std::to_string(rows) + "x" + std::to_string(cols);
      g = host_build ? gapkit::BuildCsr(gapkit::GenerateGrid(rows, cols, 0.15, 0.02, seed), false, true)
                     : gapkit::GenerateGridOnDevice(rows, cols, 0.15, 0.02, seed);
    } else {
      const bool is_kron = kron >= 0;
      const int scale = static_cast<int>(is_kron ? kron : urand);
      const gapkit::GenSpec spec{is_kron ? gapkit::GenKind::kKronecker : gapkit::GenKind::kUniformRandom, scale,
                                 static_cast<int>(degree), seed};
      const bool perm = is_kron && permute;
      name = (is_kron ? "kron" : "urand") + std::to_string(scale);
      if (host_build) {
        gapkit::EdgeList el = is_kron ? gapkit::GenerateKronecker(spec) : gapkit::GenerateUniform(spec);
        if (perm) gapkit::PermuteIds(el, scale, seed);
        g = gapkit::BuildCsr(el, false, true);
      } else {
        g = gapkit::GenerateOnDevice(spec, perm);
      }
    }
    if (bc) {  // gapkit.cc:99-121 with the bc row of the plan
      if (trials < 1 || per_trial < 1) throw gapkit::ConfigError("bc needs at least one trial and one source");
      std::string failure;
      std::vector<gapkit::BcTrial> tr =
          gapkit::RunBetweenness(g, static_cast<int>(trials), static_cast<int>(per_trial), seed, verify, &failure);
      bool all_ok = true;
      double dev = 0;
      for (const auto& t : tr) {
        all_ok &= !t.verified.has_value() || *t.verified;
        dev += t.device_ms;
      }
      if (!output.empty()) {
        std::ofstream out(output);
        if (!out) throw gapkit::ConfigError("cannot open output file: " + output);
        gapkit::WriteBcCsv(out, name, tr);
      } else {
        gapkit::WriteBcCsv(std::cout, name, tr);
      }
      std::printf("%s: n=%lld arcs=%lld bc trials=%zu x %lld sources, mean %.3f ms device per trial%s\n",
                  name.c_str(), static_cast<long long>(g.num_nodes()), static_cast<long long>(g.num_edges()),
                  tr.size(), per_trial, dev / tr.size(),
                  verify ? (all_ok ? ", all verified" : (", VERIFY FAILED: " + failure).c_str()) : "");
      return verify && !all_ok ? 1 : 0;
    }
    gapkit::BenchPlan plan;  // gapkit.cc:99-121
    plan.trials = static_cast<int>(trials);
    plan.source_seed = seed;
    plan.model = model;
    plan.peak_gbs = peak_gbs;
    if (fixed >= 0) {
      if (fixed >= g.num_nodes()) throw gapkit::ConfigError("-r source out of range");
      if (g.host_ready() && g.out_degree(static_cast<gapkit::NodeId>(fixed)) == 0)
        throw gapkit::ConfigError("-r source has zero out-degree");
      plan.fixed_source = static_cast<gapkit::NodeId>(fixed);
    }
    gapkit::BenchReport report = gapkit::RunBenchmark(g, plan, verify, name);
    if (!output.empty()) {
      std::ofstream out(output);
      if (!out) throw gapkit::ConfigError("cannot open output file: " + output);
      gapkit::WriteCsv(out, report, plan);
    } else {
      gapkit::WriteCsv(std::cout, report, plan);
    }
    std::printf("%s: n=%lld arcs=%lld trials=%d hmean %.2f GTEPS (device time)%s\n", name.c_str(),
                static_cast<long long>(g.num_nodes()), static_cast<long long>(g.num_edges()), plan.trials,
                report.HmeanDeviceGteps(), verify ? (report.AllVerified() ? ", all verified" : ", VERIFY FAILED") : "");
    return verify && !report.AllVerified() ? 1 : 0;
  } catch (const gapkit::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
