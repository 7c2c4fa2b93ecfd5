"""Kernel share table from an `ncu --metrics gpu__time_duration.sum --csv` launch list (tooling)."""
import collections, csv, re, sys
path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = re.sub(r"^void ", "", r[ki]).replace("tmvn::<unnamed>::", "").replace("tmvn::", "")
        name = re.sub(r"\(.*$", "", name)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
tot = sum(v[1] for v in agg.values())
print(title)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / tot * 100:6.2f}%  {v[0]:5d} launches  avg {v[1] / v[0]:9.2f} us  {k}")
