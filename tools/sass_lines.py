"""Aggregate ncu per-instruction stall samples by CUDA source line.

    python tools/sass_lines.py <report.ncu-rep> <kernel-substring> <cubin> [top]

The cubin must be built from the same source with -lineinfo (nvdisasm -g maps offsets)."""
import csv, io, re, subprocess, sys
from collections import Counter

rep, kname, cubin = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
m, cur, inside = {}, None, False
for l in sass:
    if l.startswith(".text.") and kname in l:
        inside = True
        continue
    if inside and l.strip().startswith(".section"):
        break
    if not inside:
        continue
    mm = re.search(r'File "([^"]+)", line (\d+)', l)
    if "//##" in l and mm:
        cur = (mm.group(1), int(mm.group(2)))
        continue
    r = re.match(r'\s+/\*([0-9a-f]+)\*/', l)
    if r:
        m[int(r.group(1), 16) // 16] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
st, ex = Counter(), Counter()
for k, r in enumerate(rows[2:]):
    st[m.get(k)] += int(r[si] or 0)
    ex[m.get(k)] += int(r[ei] or 0)
tot = sum(st.values())
srcs = {}
for key, s in st.most_common(top):
    if key is None:
        print(f"{100 * s / tot:5.1f}%  ?")
        continue
    f, line = key
    if f not in srcs:
        srcs[f] = open(f).read().splitlines()
    txt = srcs[f][line - 1].strip()[:80]
    print(f"{100 * s / tot:5.1f}%  exec {ex[key]:>11}  {f.split('/')[-1]}:{line}: {txt}")
