"""Aggregate an .ncu-rep's per-SASS counters by CUDA source line (needs -lineinfo)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
lines = [r for r in rows[hi + 1:] if len(r) > max(ie, ss) and r[0] not in ("", "Line No")]
tot_i = sum(float(r[ie] or 0) for r in lines if r[ie] not in ("-", ""))
tot_s = sum(float(r[ss] or 0) for r in lines if r[ss] not in ("-", ""))
def f(v):
    return float(v) if v not in ("-", "") else 0.0
print(f"total warp-instructions {tot_i:.0f}")
for r in sorted(lines, key=lambda r: -f(r[ie]))[:top]:
    print(f"L{r[0]:>4} inst {f(r[ie]) / tot_i * 100:5.1f}%  stall {f(r[ss]) / tot_s * 100:5.1f}%  {r[1].strip()[:90]}")
