"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel share."""
import collections, csv, sys

rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows))
h = r[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for row in r[1:]:
    name = row[ki].split("(")[0].replace("void ", "").replace("ffwd::<unnamed>::", "")
    if not name.startswith(("pool", "logits", "pooled", "gemm", "topk", "plan", "up_proj", "down_proj",
                            "rmsnorm", "rope", "allreduce", "hidden", "column")):
        name = "other (torch: init / residual copy)"
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(row[ui], 1e-6)
    tot[name] += float(row[vi].replace(",", "")) * scale
    cnt[name] += 1
ours = {k: v for k, v in tot.items() if not k.startswith("other")}
s = sum(ours.values())
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share of ours':>14s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    share = f"{100 * v / s:6.2f}%" if k in ours else "-"
    print(f"{k:40s} {cnt[k]:8d} {v:10.3f} {share:>14s}")
print(f"{'ours total':40s} {sum(cnt[k] for k in ours):8d} {s:10.3f}")
