"""Stall reasons aggregated by execution-count class (a proxy for code
region: staging loop, per-record loop, leaf loop ...) from an ncu source CSV
(ncu -i rep --page source --csv --print-source sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
cut = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
rows = rows[: cut[1]] if len(cut) > 1 else rows  # first kernel only
hdr = rows[1]
ie = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(r) for r in reasons]
agg = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
for r in rows[2:]:
    if len(r) <= max(idx):
        continue
    if not (r[ie] or "0").isdigit():
        continue
    ex = int(r[ie] or 0)
    for name, i in zip(reasons, idx):
        v = int(r[i] or 0)
        agg[ex][name] += v
        tot[name] += v
grand = sum(tot.values())
print("total", {k[6:]: round(100 * v / grand, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
top = sorted(agg.items(), key=lambda x: -sum(x[1].values()))[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for ex, d in top:
    s = sum(d.values())
    print(f"exec={ex:>10d} {100 * s / grand:5.1f}%  " +
          " ".join(f"{k[6:]}={100 * v / grand:.1f}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:5] if v))
