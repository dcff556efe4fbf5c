"""Per-launch kernel times from an `ncu --metrics gpu__time_duration.sum --csv` log.

    python tools/launch_times.py <launches.csv> [name-regex]"""
import csv, re, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for r in rows:
    n = re.sub(r"\(.*", "", r[4]).replace("void ", "")
    if pat is None or pat.search(n):
        print(f"{n:40s} {float(r[14]) / 1e3:9.1f} us")
