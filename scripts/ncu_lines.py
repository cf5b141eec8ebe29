"""Per-CUDA-source-line instruction and stall shares from an ncu report.

usage: python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [min_pct]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hk = next(k for k, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[hk]
ex = h.index("Instructions Executed")
si = next(i for i, x in enumerate(h) if "Warp Stall Sampling (All" in x)
agg = {}
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
for r in rows[hk + 1:]:
    if len(r) > ex and r[0].isdigit():  # source-line rows carry the per-line aggregates
        a = agg.setdefault((int(r[0]), r[1]), [0.0, 0.0])
        a[0] += num(r[ex])
        a[1] += num(r[si])
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot:.0f}, stall samples {ts:.0f}")
for (ln, src), (e, s) in sorted(agg.items()):
    if 100 * e / tot >= minp or 100 * s / ts >= minp:
        print(f"{ln:5d} {100 * e / tot:5.1f}% inst {100 * s / ts:5.1f}% stall  {src.strip()[:80]}")
