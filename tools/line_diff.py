"""Per-source-line difference of two ncu --set full captures of the same
kernel stopped at different barriers (GK_STOP_AFTER): what one phase adds.

    python tools/line_diff.py A.ncu-rep B.ncu-rep <lib.so> [column] [top]

column: "Instructions Executed" (default) or "Warp Stall Sampling (All Samples)".
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def per_line(rep, lib, col, kname="bfs_persistent"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the page holds one section per function ("Kernel Name", name / header / rows)
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    sec = next(i for i in starts[:-1] if kname in rows[i][1])
    h = rows[sec + 1]
    ia, ic = h.index("Address"), h.index(col)
    data = [r for r in rows[sec + 2:starts[starts.index(sec) + 1]] if r and r[ia].startswith("0x")]
    base = min(int(r[ia], 16) for r in data)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
        dis = ""
        for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):
            t = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
            if kname in t:
                dis = t
                break
    in_k, line, off2line = False, None, {}
    for l in dis.splitlines():
        if l.startswith("//---") and ".text." in l:
            in_k = kname in l
            continue
        if not in_k:
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2line[int(m.group(1), 16)] = line
    agg = collections.Counter()
    for r in data:
        agg[off2line.get(int(r[ia], 16) - base, "?")] += float(r[ic] or 0)
    return agg


def main():
    a, b, lib = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3])
    col = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    A, B = per_line(a, lib, col), per_line(b, lib, col)
    diff = {k: B[k] - A.get(k, 0) for k in B}
    tot = sum(diff.values())
    print(f"{col}: total difference {tot:.4g}")
    for k, v in sorted(diff.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v / tot * 100:6.2f}%  {v:12.4g}  {k}")


if __name__ == "__main__":
    main()
