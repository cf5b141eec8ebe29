"""Hot SASS lines of one kernel from an ncu --set full report (source page):
top lines by warp-stall samples with their dominant stall reasons, and the
kernel's stall totals.  usage: python scripts/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
j = next((k for k in range(i + 1, len(lines)) if lines[k].startswith('"Kernel Name"')), len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:j]))))
stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0 for c in stall_cols}
S = 0
for r in rows:
    for c in stall_cols:
        try:
            tot[c] += int(r[c])
        except ValueError:
            pass
    try:
        S += int(r["Warp Stall Sampling (All Samples)"])
    except ValueError:
        pass
print(f"total samples {S}")
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:22s} {v:8d} {100.0 * v / max(S, 1):5.1f}%")
def samp(r):
    try:
        return int(r["Warp Stall Sampling (All Samples)"])
    except ValueError:
        return 0
for idx, r in enumerate(rows):
    r["_i"] = idx
for r in sorted(rows, key=samp, reverse=True)[:top]:
    st = sorted(((int(r[c]) if r[c].isdigit() else 0, c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{r['_i']:5d} {samp(r):6d} {r['Instructions Executed']:>9s} {r['Source'].strip()[:60]:60s} "
          + " ".join(f"{n}:{v}" for v, n in st if v))
