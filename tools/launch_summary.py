"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
skip = [k for k in agg if "k_trsv2" in k]  # EXACT solve of the DC point (setup)
tot = sum(v[1] for k, v in agg.items() if k not in skip)
print("| kernel | launches | total ms | share (excl. setup DC solve) | avg ms |")
print("|---|---|---|---|---|")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    share = "setup" if k in skip else f"{ms / tot:.3f}"
    print(f"| `{k}` | {c} | {ms:.2f} | {share} | {ms / c:.4f} |")
