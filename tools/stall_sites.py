"""Top stall sites of one kernel in an ncu report, with the enclosing source line of the
given file (inlined helpers such as mbarrier waits are attributed to their caller).

    python tools/stall_sites.py <report.ncu-rep> <mangled-kernel-substring> <cubin> <file.cu> [top]
"""
import csv, io, re, subprocess, sys
rep, kname, cubin, fname = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 15
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
inside, seq, cur, last = False, [], None, None
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
        cur = (mm.group(1).split('/')[-1], int(mm.group(2)))
        if cur[0] == fname:
            last = cur[1]
        continue
    r = re.match(r'\s+/\*([0-9a-f]+)\*/\s+(.*)', l)
    if r:
        seq.append((cur, last, r.group(2)[:50]))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
st = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[st[0]]
d = [r for r in rows[st[0] + 1:(st[1] - 1 if len(st) > 1 else None)] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[si]) for r in d)
from collections import Counter
by = Counter()
for k, r in enumerate(d):
    by[seq[k][1]] += int(r[si])
src = open([l for l in open("/dev/null")] and "" or next(
    re.search(r'File "([^"]+)"', l).group(1) for l in sass if f'/{fname}"' in l)).read().splitlines()
for line, v in by.most_common(top):
    print(f"{100 * v / tot:5.1f}%  {fname}:{line}: {src[line - 1].strip()[:90] if line else '?'}")
