"""Print an ncu --csv metrics log as one row per launch (kernel, metric columns)."""
import csv, sys
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows))
h = r[0]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launches, metrics = {}, []
for row in r[1:]:
    key = (int(row[ii]), row[ki].split("(")[0].replace("void ", "").replace("ffwd::<unnamed>::", "")[-36:])
    launches.setdefault(key, {})[row[mi]] = row[vi]
    if row[mi] not in metrics:
        metrics.append(row[mi])
short = [m.split("__")[1][:18] if "__" in m else m[:18] for m in metrics]
print(f"{'id':>4} {'kernel':36s} " + " ".join(f"{s:>18s}" for s in short))
for (i, k), m in sorted(launches.items()):
    print(f"{i:4d} {k:36s} " + " ".join(f"{m.get(x, ''):>18s}" for x in metrics))
