"""Per-kernel-class summary of an ncu `--cache-control none` duration capture
(warm caches, serialised launches):

    ncu --profile-from-start off --cache-control none --clock-control none \
        --metrics gpu__time_duration.sum --csv --log-file warm.csv python scripts/traffic_step.py
    python scripts/warm_summary.py warm.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Value", "Grid Size")}
g = collections.OrderedDict()
for r in rows[i + 1:]:
    if len(r) != len(h):
        continue
    m = re.search(r"::(\w+)(<[^(]*>)?\(", r[ix["Kernel Name"]])
    n = (m.group(1) + (m.group(2) or "").replace(" ", "")) if m else r[ix["Kernel Name"]][:40]
    g.setdefault((n, r[ix["Grid Size"]]), []).append(float(r[ix["Metric Value"]].replace(",", "")))
tot = sum(sum(v) for v in g.values())
print("| kernel | grid | launches | avg us | share |\n|---|---|---:|---:|---:|")
for k, v in sorted(g.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {k[0]} | {k[1]} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
print(f"\ntotal {tot / 1e3:.1f} us")
