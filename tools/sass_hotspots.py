"""Map ncu per-SASS stall samples to source lines.

    python tools/sass_hotspots.py <report.ncu-rep> <lib.so> [kernel_substr] [top]

Uses `ncu --page source --print-source sass` for the samples and
`nvdisasm -g` (line info from -lineinfo) on the cubin inside <lib.so>.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, lib = sys.argv[1], os.path.abspath(sys.argv[2])
    kname = sys.argv[3] if len(sys.argv) > 3 else "bfs_persistent"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # one section per function ("Kernel Name", name / header / rows)
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    sec = next((i for i in starts[:-1] if kname in rows[i][1]), None)
    if sec is None:
        h, data = rows[1], rows[2:]
    else:
        h = rows[sec + 1]
        data = rows[sec + 2:starts[starts.index(sec) + 1]]
    data = [r for r in data if r and r[h.index("Address")].startswith("0x")]
    ia, iw = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    base = min(int(r[ia], 16) for r in data)
    samples = {int(r[ia], 16) - base: (float(r[iw] or 0), {h[i]: float(r[i] or 0) for i in stall_cols})
               for r in data}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
        dis = ""
        for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):
            t = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                               text=True).stdout
            if kname in t:
                dis = t
                break
    # walk the kernel's section; track the current "//## File ..., line N" annotation
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
    agg = collections.defaultdict(lambda: [0.0, collections.Counter()])
    tot = 0.0
    for off, (s, st) in samples.items():
        key = off2line.get(off, "?")
        agg[key][0] += s
        agg[key][1].update(st)
        tot += s
    print(f"total samples {tot:.0f}")
    for key, (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        main_st = ", ".join(f"{k[6:]}={v / s * 100:.0f}%" for k, v in st.most_common(3) if v > 0)
        print(f"{s / tot * 100:6.2f}%  {key:28s} {main_st}")


if __name__ == "__main__":
    main()
