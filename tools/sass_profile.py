"""Per-opcode instruction and stall-sample shares of one kernel in an .ncu-rep (no GPU).
usage: sass_profile.py REP KERNEL_REGEX [N]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
ie, si, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
stall_cols = [j for j, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
ops, st = collections.Counter(), collections.Counter()
reasons = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ie or r[0] == h[0]:
        if r and r[0] == "Address":
            break  # next kernel instance
        continue
    try:
        n = float(r[ie] or 0)
    except ValueError:
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = ".".join(op.split(".")[:2])
    ops[op] += n
    st[op] += float(r[si] or 0)
    for j in stall_cols:
        reasons[h[j]] += float(r[j] or 0)
tot, stot = sum(ops.values()) or 1, sum(st.values()) or 1
print(f"instructions executed (warp): {tot:.0f}")
for op, n in ops.most_common(ntop):
    print(f"  {op:18s} inst {n / tot * 100:5.1f}%   stall samples {st[op] / stot * 100:5.1f}%")
rt = sum(reasons.values()) or 1
print("stall reasons:", ", ".join(f"{k[6:]} {v / rt * 100:.1f}%" for k, v in reasons.most_common(8)))
