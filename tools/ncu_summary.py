#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.md>   # --set full capture
    python tools/ncu_summary.py launches <launches.csv> <out.md>  # gpu__time_duration list
"""
import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "tmem pipe inst %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
]


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", "",
             "One row per captured launch (cold-cache, serialised replay; compare shares, not "
             "absolute times, with bench.py).", ""]
    cols = [(m, n) for m, n in FULL_METRICS if m in h]
    lines.append("| kernel | " + " | ".join(n for _, n in cols) + " |")
    lines.append("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")])
        vals = []
        for m, _ in cols:
            v, u = r[h.index(m)], units[h.index(m)]
            vals.append(f"{v} {u}".strip())
        lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    seq = [(re.sub(r"\(.*", "", r[4]).replace("void ", "").strip(), r[6], float(r[14]) / 1e3)
           for r in rows]
    # one steady-state round: from a quantiser launch (end of compress) to the next one,
    # taking the last such segment with exactly one fused outer-update launch (the device-
    # resident rounds; the host-pipeline rounds update in tensor groups)
    qp = [i for i, (n, _, _) in enumerate(seq) if n.startswith("dlx::k_quant_pack")]
    rnd = seq
    for a, b in reversed(list(zip(qp, qp[1:]))):
        seg = seq[a + 1:b + 1]
        if sum(1 for n, _, _ in seg if n.startswith("dlx::k_o5<") or n.startswith("dlx::k5")) == 1:
            rnd = seg
            break
    agg = OrderedDict()
    for n, s, t in rnd:
        k = (n, s)
        c, tt = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, tt + t)
    total = sum(t for _, _, t in rnd)
    main = sum(t for n, s, t in rnd if s == rnd[-1][1])
    lines = [f"# Launch list of one steady-state round (`{path.split('/')[-1]}`)", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`bench.py --steps 2 --warmup 3`; launches from one round's quantiser to the next "
             "(effective rank + outer update of round t, compress of round t+1). Serialised "
             "and cold-cache: use the shares.", "",
             f"Sum of kernel times: {total:.1f} us ({main:.1f} us on the main stream).", "",
             "| kernel | stream | launches | total us | share |", "|---|---|---|---|---|"]
    for (n, s), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{n}` | {s} | {c} | {t:.1f} | {100 * t / total:.1f} % |")
    lines += ["", "Sequence:", "", "```"]
    lines += [f"{n:40s} stream {s:>3s} {t:9.1f} us" for n, s, t in rnd]
    lines.append("```")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
