"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total/mean device time and share of the total."""
import csv, sys, re, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i0 + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    name = re.sub(r"<unnamed>::|ds::|::<unnamed>", "", name)[:70]
    v = float(r[vi].replace(",", ""))
    unit = hdr  # values are in the unit of the column (ns or us); normalised below
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
print(f"| kernel | launches | total | mean | share |\n|---|---:|---:|---:|---:|")
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"| `{k}` | {n} | {v:.1f} | {v / n:.2f} | {100 * v / tot:.1f}% |")
print(f"\ntotal device time over {sum(n for n, _ in agg.values())} launches: {tot:.1f} (unit of the csv: see header)")
