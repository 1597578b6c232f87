"""Summaries of tools/prof_round.sh outputs (gpurun_out/) for profiles/rNN/:
per-launch DRAM traffic of bfs_persistent over 16 sources (+ the parent
memset), profiles/ncu_traffic.json for bench.py, the full-capture metrics.

    python tools/prof_summarize.py profiles/r01
"""
import collections
import csv
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
        "ns": 1e-6, "us": 1e-3, "ms": 1}
FULL_METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
                "l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,"
                "smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,"
                "launch__block_size,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,"
                "lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,"
                "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,"
                "lts__t_sectors_srcunit_tex_op_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,"
                "smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,"
                "smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,"
                "smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_sample_count,smsp__inst_executed.sum")


def main():
    dst = sys.argv[1]
    commit = subprocess.run(["git", "log", "--oneline", "-1"], capture_output=True, text=True, cwd=ROOT).stdout.split()[0]
    srcs = [l.split()[1] for l in open(os.path.join(OUT, "one16.log")) if l.startswith("src")]
    rows = [r for r in csv.reader(open(os.path.join(OUT, "traffic16.csv"))) if len(r) > 10]
    h = rows[0]
    iid, im, iv, iu = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", "")) * MULT.get(r[iu], 1)
    n = 1 << 27
    out = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
           "#   -k regex:bfs_persistent python tools/ncu_one.py --config kron27 --runs 16   (first 16 picked sources)",
           f"# kernel of commit {commit}.  parent := -1 is a cudaMemsetAsync ahead of each launch",
           f"# ({4 * n / 1e9:.3f} GB written, not in these kernel counters).",
           "# source        ms(ncu, cold, serialised)   DRAM read GB   DRAM write GB   traffic GB"]
    tot = []
    for s, d in zip(srcs, per.values()):
        r, w, t = d["dram__bytes_read.sum"] / 1e9, d["dram__bytes_write.sum"] / 1e9, d["gpu__time_duration.sum"]
        tot.append(r + w)
        out.append(f"{s:>12} {t:11.3f} {r:15.3f} {w:15.3f} {r + w:12.3f}")
    m = statistics.mean(tot)
    out.append(f"# mean kernel traffic per launch: {m:.3f} GB over {len(tot)} launches; "
               f"+ {4 * n / 1e9:.3f} GB memset = {m + 4 * n / 1e9:.3f} GB per BFS")
    open(os.path.join(dst, "ncu_traffic16_kron27.txt"), "w").write("\n".join(out) + "\n")
    json.dump({"config": "kron27", "kernel": "bfs_persistent + parent memset", "sources": "first 16 of the 64 picked",
               "dram_bytes_per_launch": int(m * 1e9 + 4 * n), "kernel_dram_bytes_per_launch": int(m * 1e9),
               "memset_bytes_per_launch": 4 * n, "commit": commit,
               "note": "mean dram__bytes_read.sum + dram__bytes_write.sum of bfs_persistent per launch over 16 "
                       "sources, plus the 4n-byte parent memset that precedes each launch inside the timed region; "
                       f"{dst}/ncu_traffic16_kron27.txt"},
              open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, "kron_full.ncu-rep"), "--page", "raw", "--metrics",
                          FULL_METRICS], capture_output=True, text=True).stdout
    lines = ["# ncu --set full --import-source on --clock-control none -k regex:bfs_persistent -s 0 -c 1",
             "#   python tools/ncu_one.py --config kron27 --runs 1   (source 13825371)",
             f"# kernel of commit {commit}; the parent memset is not part of this launch"]
    for l in raw.splitlines():
        p = l.split()
        if len(p) >= 3 and "__" in p[0]:
            lines.append(f"{p[0]:<62} {p[-2]:>18} {p[-1]}")
    open(os.path.join(dst, "ncu_full_bfs_persistent_kron27.txt"), "w").write("\n".join(lines) + "\n")
    subprocess.run(["cp", os.path.join(OUT, "launches.csv"), os.path.join(dst, "ncu_launches_bench_kron27.csv")])
    print("\n".join(out[-3:]))
    print("\n".join(lines[3:12]))


if __name__ == "__main__":
    main()
