#!/usr/bin/env python
"""bench.py -- BFS GTEPS (harmonic mean over sources) + % of HBM roofline.

Default workload = BASELINE config 3 (the north_star's 1-GPU target): a
Kronecker graph of 2^27 vertices, edge factor 16, initiator .57/.19/.19,
seeded (24601), vertex IDs permuted, symmetrized/deduplicated, generated and
built on the device bit-identically to the reference generator + BuildCsr.
A "step" is one BFS (gk_bfs, the C-ABI replacement of gapkit::Bfs,
bfs.hpp:117) from the next of PickSources(g, K, seed) (source_picker.hpp:47).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config kron27|urand27|kron16|grid4900|kron30|kronS|urandS]

value     : harmonic mean over the K steps of m_cc(s)/t_dev(s) (GTEPS), t_dev the
            CUDA-event time of the traversal kernel, graph resident in HBM.
e2e       : same metric through the C ABI with the parent array returned to a
            pinned host buffer (D2H inside the timed region), host wall clock.
roofline  : algorithmic bytes B_sec (evaluated per source from
            exact depths + the executed direction schedule) / t_dev vs the
            measured HBM copy bandwidth (MEASURED_PEAKS.json).
cpu_baseline : the reference's own OpenMP Bfs (oracle/_ref/libgapref.so, the
            unmodified headers) on the box's host cores, bounded sample.
N > 1     : one process per GPU (torchrun).  Default (--multi sharded): the
            1D vertex-partitioned traversal of ONE graph:
            one persistent kernel per rank, the level loop on the device,
            bitmap exchanges over NVLink peer memory, device-side cross-rank
            barriers; strong scaling, step time = max over ranks; the line
            adds the NVLink fraction.  --multi replicas: every rank holds the
            whole graph and runs its own sources (weak scaling).
            --emulate-ranks P at N=1: the sharded kernel with P ranks in one
            launch on one GPU (its overhead against the single-device kernel).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "kron27": dict(kind="kron", scale=27, degree=16, permute=True,
                   workload="BASELINE config 3: Kronecker 2^27 vertices, edge factor 16, A/B/C=.57/.19/.19, "
                            "permuted IDs, symmetrized+deduplicated, int32 IDs, CSR"),
    "urand27": dict(kind="urand", scale=27, degree=16, permute=False,
                    workload="BASELINE config 2: uniform random 2^27 vertices, 2^31 generated edges, "
                             "symmetrized+deduplicated, CSR"),
    "kron16": dict(kind="kron", scale=16, degree=16, permute=True,
                   workload="BASELINE config 1: Kronecker 2^16 vertices, edge factor 16, permuted"),
    "kron30": dict(kind="kron", scale=30, degree=16, permute=True,
                   workload="BASELINE config 5's graph: Kronecker 2^30 vertices, edge factor 16, permuted, "
                            "symmetrized+deduplicated (34.0 G arcs, 145 GB CSR) on ONE B200"),
    "grid4900": dict(kind="grid", rows=4900, cols=4900, p_delete=0.15, p_diag=0.02,
                     workload="BASELINE config 4: 4900x4900 4-neighbour grid, 15% edges deleted, "
                              "2% diagonal shortcuts"),
}
SEED = 24601
# One metric string for both arms (ours and --impl reference): the driver
# pairs the two lines by it.  The HBM-roofline half of BASELINE.json's metric
# is the line's "roofline" object.
METRIC = "BFS GTEPS (harmonic mean over sources)"
L2_NOTE = "inputs larger than L2 (CSR %.1f GB vs 126 MB L2)"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse_config(name: str) -> dict:
    if name in CONFIGS:
        return dict(CONFIGS[name], name=name)
    for kind in ("kron", "urand"):
        if name.startswith(kind) and name[len(kind):].isdigit():
            sc = int(name[len(kind):])
            return dict(kind=kind, scale=sc, degree=16, permute=(kind == "kron"), name=name,
                        workload=f"{kind} 2^{sc} vertices, edge factor 16" + (", permuted" if kind == "kron" else ""))
    raise SystemExit(f"unknown config {name}")


def line_config(cfg: dict, n: int, arcs: int, K: int) -> dict:
    """The workload both arms print (identical keys and values)."""
    csr = arcs * 4 + n * 8
    l2 = (L2_NOTE % (csr / 1e9)) if csr > 126e6 else \
        f"graph L2-resident (CSR {csr / 1e6:.0f} MB < 126 MB L2), as a loaded graph stays between GAP trials"
    return {"workload": cfg["workload"], "name": cfg["name"], "n": int(n), "arcs": int(arcs), "seed": SEED,
            "sources": K, "alpha": 15, "beta": 18, "l2": l2}


def cpp_shim_e2e(cfg: dict, trials: int, n: int):
    """e2e through the C++ surface: the host CLI (`gapkit_b200 bfs`, built on
    host/gapkit_b200/bfs.hpp's `gapkit::Bfs(g, src)`) builds the same graph
    and times `trials` calls on the first sources of the same picker, each
    returning a fresh ParentArray (std::vector, pageable) -- the CSV's
    elapsed_seconds, host wall clock per call as benchmark.hpp:153-193 times
    it.  The call also counts m_cc (one extra pass), so this is slightly
    conservative.  None when the CLI is not built or the config has no flag."""
    exe = os.path.join(ROOT, "paper_1508_03619_b200", "host", "bin", "gapkit_b200")
    if cfg["kind"] == "kron":
        gflags = ["-g", str(cfg["scale"])] + ([] if cfg.get("permute", True) else ["--no-permute"])
    elif cfg["kind"] == "urand":
        gflags = ["-u", str(cfg["scale"])]
    elif cfg["kind"] == "grid":
        gflags = ["--grid", f"{cfg['rows']}x{cfg['cols']}"]
    else:
        return None
    if not os.path.exists(exe):
        return {"value": None, "note": "host CLI not built (make host)"}
    out = os.path.join("/tmp", f"gk_cpp_e2e_{os.getpid()}.csv")
    cmd = [exe, "bfs"] + gflags + ["-k", str(cfg.get("degree", 16)), "-n", str(trials + 2), "--seed", str(SEED),
                                   "--no-model", "-o", out]
    try:
        # without the CPU reference's OpenMP binding (set for cpu_reference
        # in main): OMP_PROC_BIND pins the CLI's master thread to one core,
        # and the host threads of the copy-out would inherit that mask
        env = {k: v for k, v in os.environ.items() if k not in ("OMP_PROC_BIND", "OMP_WAIT_POLICY")}
        subprocess.run(cmd, check=True, capture_output=True, timeout=600, env=env)
        with open(out) as f:
            rows = [r.split(",") for r in f.read().splitlines()[1:] if r.startswith("bfs,")][2:]
        os.unlink(out)
    except Exception as ex:  # reported, never required
        return {"value": None, "note": f"host CLI failed: {ex}"}
    g_e = [int(r[7]) / float(r[4]) / 1e9 for r in rows if float(r[4]) > 0]
    return {"value": hmean(g_e), "unit": "GTEPS", "trials": len(g_e),
            "per_call_ms": [round(float(r[4]) * 1e3, 2) for r in rows], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * n,
            "note": "gapkit::Bfs(g, src) through the host CLI: each call allocates a std::vector ParentArray "
                    "and copies the result into it (pageable), host wall clock per call (CSV elapsed_seconds), "
                    "sources 3.. of the same picker (the first two calls are warm-up: CUDA-graph instantiation, pool "
                    "growth, pinned stage allocation); graph built by the CLI, untimed"}


def hmean(xs):
    xs = [x for x in xs if x > 0]
    return len(xs) / sum(1.0 / x for x in xs) if xs else 0.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"gk_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                r = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for bit, name in REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def build_graph(cfg, device):
    from paper_1508_03619_b200 import DeviceGraph
    t0 = time.time()
    if cfg["kind"] == "grid":
        g = DeviceGraph.grid(cfg["rows"], cfg["cols"], cfg["p_delete"], cfg["p_diag"], SEED, device=device)
    else:
        g = DeviceGraph.generate(cfg["kind"], cfg["scale"], cfg["degree"], SEED, permute=cfg["permute"],
                                 device=device)
    return g, time.time() - t0


def host_ref_graph(g):
    """Download the device CSR straight into the reference's CsrGraph vectors
    (public constructor, graph.hpp:30-45)."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O
    R = O.RefLib()
    po, pn, pio, pin = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    h = R.L.gkr_graph_alloc(g.n, g.m, 0, C.byref(po), C.byref(pn), C.byref(pio), C.byref(pin))
    g.download_into(po.value, pn.value)
    off = np.frombuffer((C.c_int64 * (g.n + 1)).from_address(po.value), np.int64).copy()
    err = C.create_string_buffer(256)
    R.L.gkr_graph_seal(h, 0, err, 256)
    return O.RefGraph(R, h), off


def cpu_reference(g, sources, warmup, budget_s, label, m_of=None):
    """Time gapkit::Bfs (the reference) on the host cores; bounded by budget_s."""
    import numpy as np
    t0 = time.time()
    rg, off = host_ref_graph(g)
    deg = np.diff(off)
    threads = rg.ref.L.gkr_max_threads()
    for s in sources[:warmup]:
        rg.bfs_timed([int(s)])
    secs, gteps, done = [], [], 0
    tstart = time.time()
    for s in sources:
        sec = float(rg.bfs_timed([int(s)])[0])
        if m_of is not None and int(s) in m_of:
            m = m_of[int(s)]
        else:
            p = rg.bfs(int(s))
            m = int(deg[p >= 0].sum()) // 2
        secs.append(sec)
        gteps.append(m / sec / 1e9)
        done += 1
        if time.time() - tstart > budget_s:
            break
    # a 1-thread row next to the all-cores one (bounded)
    rg.ref.L.gkr_set_threads(1)
    one, t1 = [], time.time()
    for s in sources:
        sec = float(rg.bfs_timed([int(s)])[0])
        m = m_of[int(s)] if m_of is not None and int(s) in m_of else int(deg[rg.bfs(int(s)) >= 0].sum()) // 2
        one.append(m / sec / 1e9)
        if time.time() - t1 > min(budget_s, 12.0):
            break
    rg.ref.L.gkr_set_threads(threads)
    return {"value": hmean(gteps), "unit": "GTEPS", "cores": threads, "kind": "reference",
            "sample": f"{label}: first {done} of the {len(sources)} picked sources, gapkit::Bfs "
                      f"(oracle/_ref, unmodified reference headers, OpenMP {threads} threads, "
                      f"OMP_WAIT_POLICY=active, OMP_PROC_BIND=spread), steady_clock per call incl. allocation",
            "one_thread": {"value": hmean(one), "unit": "GTEPS", "cores": 1,
                           "sample": f"first {len(one)} of the same sources, OpenMP 1 thread"},
            "mean_ms": 1e3 * sum(secs) / max(len(secs), 1), "setup_s": round(tstart - t0, 2)}


def reference_arm(args, cfg, K, W):
    """--impl reference: the UNMODIFIED reference on the host cores, nothing
    of ours on the path.  Graph: the reference's generator (or the grid),
    the ID permutation and a 64-bit BuildCsr on the host (oracle/ref_bench.cc,
    pinned byte-identical to BuildCsr); sources: PickSources
    (source_picker.hpp:47-54); trials: RunBenchmark's BFS loop
    (benchmark.hpp:178-185) around gapkit::Bfs.  libgk_bfs.so is never loaded."""
    from oracle import oracle as O
    R = O.RefLib()
    t0 = time.time()
    if cfg["kind"] == "grid":
        rg = R.bench_graph("grid", seed=SEED, rows=cfg["rows"], cols=cfg["cols"], p_delete=cfg["p_delete"],
                           p_diag=cfg["p_diag"])
    else:
        rg = R.bench_graph(cfg["kind"], cfg["scale"], cfg["degree"], SEED, permute=cfg["permute"])
    build_s = time.time() - t0
    sources = rg.pick_sources(K, SEED)
    if W:
        rg.trials((list(sources) * (W // max(K, 1) + 1))[:W])
    secs, mcc = rg.trials(sources)
    value = hmean([m / t / 1e9 for m, t in zip(mcc, secs)])
    threads = R.L.gkr_max_threads()
    sample = (f"{cfg['name']}: all {K} picked sources, gapkit::Bfs (unmodified reference headers, "
              f"oracle/_ref), OpenMP {threads} threads, OMP_WAIT_POLICY=active, OMP_PROC_BIND=spread; "
              f"graph built on the host (reference generator + 64-bit BuildCsr) in {build_s:.0f} s")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * statistics.mean(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded generator, no dataset)",
            "config": line_config(cfg, rg.n, rg.m, K),
            "run": {"host_cpu": cpu_model(), "nproc": os.cpu_count(), "host_build_s": round(build_s, 1)},
            "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_sharded(args, cfg, rank, world, local, dist):
    """N GPUs, one graph, one persistent kernel per rank (dist.ShardedBfs:
    1D vertex partition, device-driven level loop, exchanges over NVLink
    peer memory); strong scaling.  --emulate-ranks P on one
    GPU runs the same kernel with P ranks in one launch (dist.ShardGroup)."""
    import numpy as np
    import torch

    from paper_1508_03619_b200 import DeviceGraph
    from paper_1508_03619_b200.dist import ShardedBfs, ShardGroup, pick_sources
    K, W = args.steps, max(args.warmup, 0)
    P = world if world > 1 else max(1, args.emulate_ranks)
    t0 = time.time()
    if world > 1:
        runner = ShardedBfs.generate(cfg["kind"], cfg["scale"], cfg["degree"], SEED, cfg["permute"], rank, world,
                                     local)
        shard = runner.shard
        off = shard.local_offsets()
        owned = (shard.lo, shard.hi)

        def degree_of(v):  # PickSources over the partition: the owner answers
            d = int(off[v - owned[0] + 1] - off[v - owned[0]]) if owned[0] <= v < owned[1] else 0
            t = torch.tensor([d], dtype=torch.int64, device="cuda")
            dist.all_reduce(t)
            return int(t.item())
    else:
        runner = ShardGroup.generate(cfg["kind"], cfg["scale"], cfg["degree"], SEED, cfg["permute"], P, local)
        offs = [sh.local_offsets() for sh in runner.shards]
        deg = np.concatenate([np.diff(o) for o in offs])

        def degree_of(v):
            return int(deg[v])
    build_s = time.time() - t0
    n = runner.n
    sources = pick_sources(degree_of, n, K, SEED)
    for s in (sources * (W // max(K, 1) + 1))[:W]:
        runner.run(s, parent=False)
    # algorithmic bytes: the single-device byte model of the same graph (rank 0, untimed)
    bsec_of = {}
    if rank == 0 and not args.no_model:
        full = DeviceGraph.generate(cfg["kind"], cfg["scale"], cfg["degree"], SEED, permute=cfg["permute"],
                                    device=local)
        full.keep_depth(True)
        for s in sources:
            r = full.bfs(s, parent=False)
            bsec_of[s] = full.byte_model(r.steps)[0]
        del full
        torch.cuda.empty_cache()
    m_of, scheds = {}, {}
    for s in sources:  # untimed: component edges
        r = runner.run(s, parent=False, counts=True)
        if world > 1:
            t = torch.tensor([r.component_edges], dtype=torch.int64, device="cuda")
            dist.all_reduce(t)
            m_of[s] = int(t.item()) // 2
        else:
            m_of[s] = r.component_edges
        scheds[s] = r.schedule
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.2)
    dev_ms, nvl = [], []
    launches0 = runner.launches()
    for s in sources:
        if dist:
            dist.barrier()
        r = runner.run(s, parent=False)
        dev_ms.append(r.device_ms)
        nvl.append(max(r.bytes_in))
    clocks = clk.stop()
    launches = runner.launches() - launches0
    e2e_s = []
    for s in sources:  # every rank's owned parents to host memory
        if dist:
            dist.barrier()
        t1 = time.perf_counter()
        runner.run(s, parent=True)
        e2e_s.append(time.perf_counter() - t1)
    if dist:
        t = torch.tensor(dev_ms + e2e_s + nvl, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = t.tolist()
        dev_ms, e2e_s, nvl = vals[:K], vals[K:2 * K], vals[2 * K:]
    arcs = _arcs_of(runner, world, dist)
    if rank != 0:
        return
    ms = [m_of[s] for s in sources]
    value = hmean([m / (t * 1e-3) / 1e9 for m, t in zip(ms, dev_ms)])
    peak, peak_src = peaks()
    roof = None
    tot_t = sum(dev_ms) * 1e-3
    nvl_gbs = sum(nvl) / tot_t / 1e9
    nvlink = {"achieved": nvl_gbs, "peak": 900.0, "unit": "GB/s", "frac": nvl_gbs / 900.0,
              "bytes_in_per_bfs_max_rank": sum(nvl) / len(nvl),
              "peak_source": "NVLink 5, 900 GB/s per direction per GPU (B200_PROFILING.md)",
              "note": "exchange bytes received per rank: all-gather of next per step + claims reduce per "
                      "top-down step" + ("" if world > 1 else "; ranks emulated on one GPU (no NVLink)")}
    if bsec_of:
        per_gpu = sum(bsec_of[s] for s in sources) / world / tot_t / 1e9  # emulated ranks share one GPU
        roof = {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s", "frac": per_gpu / peak,
                "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": sum(bsec_of[s] for s in sources) / len(sources) / world,
                "note": "per-GPU share (B_sec / N) of the single-device byte model over the sharded step time",
                "kernel": "bfs_sharded (one persistent launch per rank per BFS)", "nvlink": nvlink}
    line = {
        "metric": METRIC,
        "value": value, "unit": "GTEPS", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": statistics.mean(dev_ms), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded generator, no dataset)",
        "config": line_config(cfg, n, arcs, K),
        "run": {"parallelism": f"1D vertex partition over {P} rank(s)" +
                (", one per GPU, exchanges over NVLink peer memory" if world > 1 else ", emulated in one launch"),
                "trial": "one persistent kernel per rank: allocation, initialisation, the level loop with "
                         "device-side cross-rank barriers -- CUDA events around all of it, max over ranks",
                "device_build_s": round(build_s, 2), "schedules": sorted(set(scheds.values()), key=len)[:4]},
        "e2e": {"value": hmean([m / t / 1e9 for m, t in zip(ms, e2e_s)]), "unit": "GTEPS",
                "h2d_bytes_per_step": 4, "d2h_bytes_per_step": 4 * n // max(world, 1),
                "note": "sharded run + each rank's owned parent array D2H (max over ranks)"},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roof,
        "nvlink": nvlink,
        "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def _arcs_of(runner, world, dist):
    import torch
    if world > 1:
        t = torch.tensor([runner.shard.m], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        return int(t.item())
    return sum(sh.m for sh in runner.shards)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="kron27")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of reference CPU BFS work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-model", action="store_true")
    ap.add_argument("--no-cpp-e2e", action="store_true", help="skip the C++ Bfs(g, src) e2e leg")
    ap.add_argument("--verbose", action="store_true", help="per-source times on stderr")
    ap.add_argument("--multi", default="sharded", choices=["sharded", "replicas"],
                    help="N>1: the 1D-partitioned traversal of one graph (default; strong scaling) or "
                         "source-parallel whole-graph replicas (weak scaling)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="N=1: run the sharded kernel with this many ranks emulated in one launch")
    args = ap.parse_args()
    # OpenMP settings for the reference CPU legs (must precede libgomp init).
    os.environ.setdefault("OMP_WAIT_POLICY", "active")
    os.environ.setdefault("OMP_PROC_BIND", "spread")
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = parse_config(args.config)
    K, W = args.steps, max(args.warmup, 0)
    if args.impl == "reference":  # rank 0 alone; no NCCL, no GPU, no libgk_bfs.so
        if rank == 0:
            print(json.dumps(reference_arm(args, cfg, K, W)), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1508_03619_b200 import PinnedBuffer

    # ---------------- our arm ----------------
    fallback = None
    if cfg["kind"] != "grid" and args.multi == "sharded" and (world > 1 or args.emulate_ranks > 0):
        from paper_1508_03619_b200.dist import ShardConnectError
        try:
            run_sharded(args, cfg, rank, world, local, dist)
            if dist:
                dist.destroy_process_group()
            return
        except ShardConnectError as ex:  # raised on every rank together (dist.ShardedBfs)
            fallback = f"sharded traversal unavailable ({ex}); ran source-parallel replicas instead"
            print(f"rank {rank}: {fallback}", file=sys.stderr, flush=True)
            import gc
            gc.collect()
    g, build_s = build_graph(cfg, local)
    sources = [int(s) for s in g.pick_sources(K, SEED + rank)]
    warm = sources[: max(W, 0)] if W <= K else (sources * (W // K + 1))[:W]
    for s in warm:
        g.bfs(s, parent=False)
    # untimed pre-pass: exact depths -> m_cc and the B_sec/B_use byte model
    m_of, bsec_of, buse_of, sched_of = {}, {}, {}, {}
    if not args.no_model:
        g.keep_depth(True)
    verified = 0
    for s in sources:
        r = g.bfs(s, parent=False, counts=True)
        m_of[s] = r.component_edges
        sched_of[s] = r.schedule
        if not args.no_model:
            bsec_of[s], buse_of[s] = g.byte_model(r.steps)
            verified += bool(g.verify(s)["ok"])  # device BFS certificate (untimed)
    g.keep_depth(False)

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.2)
    if dist:
        dist.barrier()
    tw0 = time.time()
    dev_ms = []
    launches0 = g.launches()
    for s in sources:
        r = g.bfs(s, parent=False)
        dev_ms.append(r.device_ms)
    launches = g.launches() - launches0
    wall = time.time() - tw0
    clocks = clk.stop()
    if args.verbose:
        for s, t in zip(sources, dev_ms):
            print(f"rank {rank} src {s}: {t:.3f} ms  m_cc {m_of[s]}  {sched_of[s][:40]}", file=sys.stderr)

    # e2e: the public batch call (gk_bfs_batch) with every source's
    # ParentArray returned to pinned host memory inside the timed region; the
    # copy of result i overlaps traversal i+1.  One-call-per-source timing
    # (gk_bfs, copy not overlapped) is reported beside it.
    pins = [PinnedBuffer(g.n), PinnedBuffer(g.n)]
    # warm-up batch over the same K sources: the handle's per-batch event
    # and error arrays grow to K here, outside the timed call
    g.bfs_batch(sources, [pins[i & 1].array for i in range(len(sources))])
    t0 = time.perf_counter()
    g.bfs_batch(sources, [pins[i & 1].array for i in range(len(sources))])
    batch_s = time.perf_counter() - t0
    e2e_s = [batch_s / len(sources)] * len(sources)
    d2h_total, d2h_packed = g.batch_d2h_bytes()
    single_s = []
    for s in sources[: min(8, len(sources))]:
        t0 = time.perf_counter()
        g.bfs(s, parent=pins[0].array)
        single_s.append(time.perf_counter() - t0)
    cpp = cpp_shim_e2e(cfg, min(8, len(sources)), g.n) if world == 1 and not args.no_cpp_e2e else None

    if dist:
        import torch
        t = torch.tensor(dev_ms, dtype=torch.float64, device="cuda")
        m = torch.tensor([m_of[s] for s in sources], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(m, op=dist.ReduceOp.SUM)
        step_ms, step_m = t.tolist(), m.tolist()
        e = torch.tensor(e2e_s, dtype=torch.float64, device="cuda")
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        e2e_step = e.tolist()
    else:
        step_ms, step_m, e2e_step = dev_ms, [m_of[s] for s in sources], e2e_s

    gteps = [m / (t * 1e-3) / 1e9 for m, t in zip(step_m, step_ms)]
    value = hmean(gteps)
    e2e_val = hmean([m / t / 1e9 for m, t in zip(step_m, e2e_step)])
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    roof = None
    if bsec_of:
        tot_b = sum(bsec_of[s] for s in sources)
        tot_t = sum(dev_ms) * 1e-3
        ach = tot_b / tot_t / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("config") == cfg["name"]:
                traffic = tj.get("dram_bytes_per_launch")
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": tot_b / len(sources),
                "b_use_frac": (sum(buse_of[s] for s in sources) / tot_t / 1e9) / peak,
                "frac_of_8TBs_nominal": ach / 8000.0,
                "kernel": ("bfs_persistent (one launch per BFS)" if launches == len(sources) else
                           f"bfs_persistent + bfs_cluster ({launches} launches for {len(sources)} BFS: "
                           "chains of tiny top-down levels run in the cluster kernel)"),
                "per": "BFS (all of its launches)"}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_reference(g, sources, 1, args.cpu_budget, cfg["name"], m_of)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "one_thread")}
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GTEPS", "cores": 0, "kind": "reference", "sample": f"unavailable: {ex}"}

    scheds = sorted(set(v if len(v) <= 48 else f"{v[:40]}...({len(v)} steps)" for v in sched_of.values()),
                    key=len)
    line = {
        "metric": METRIC,
        "value": value, "unit": "GTEPS", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": statistics.mean(step_ms), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded generator, no dataset)",
        "config": line_config(cfg, g.n, g.m, K),
        "run": {"parallelism": "single GPU" if world == 1 else
                f"{world} source-parallel replicas (whole graph per GPU, no data-path collective)"
                + (f" -- {fallback}" if fallback else ""),
                "trial": "one gk_bfs: pool allocation of the result and all scratch, their initialisation, "
                         "the traversal kernel, scratch release -- CUDA events around all of it",
                "device_build_s": round(build_s, 2), "timed_region_wall_s": round(wall, 4),
                "schedules": scheds[:4], "mean_m_cc": statistics.mean(step_m),
                "verified": (f"{verified}/{len(sources)} sources pass the device BFS certificate "
                             "(depths exact, parents valid)") if not args.no_model else "not run"},
        "e2e": {"value": e2e_val, "unit": "GTEPS", "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": d2h_total / len(sources),
                "result_bytes_per_step": 4 * g.n, "compact_sources": d2h_packed,
                "one_call_per_source": hmean([m_of[s] / t / 1e9 for s, t in zip(sources, single_s)]),
                "note": "gk_bfs_batch over the K sources, every source's parent array copied to pinned host "
                        "memory inside the timed region (copy of result i overlaps traversal i+1); "
                        "compact_sources of them travel as reached bitmap + packed parents and are "
                        "expanded into the full ParentArray by host threads inside the timed region; "
                        "one_call_per_source = gk_bfs per source without overlap (first 8 sources); graph "
                        "resident (uploaded once, untimed, as the reference harness builds it untimed); "
                        "the per-step input is the 4-byte source id (a kernel argument)",
                "cpp_shim": cpp},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roof,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
