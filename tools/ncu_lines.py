"""Aggregate ncu source-page warp-stall samples per source line (tooling)."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
cur_file = cur_line = cur_src = None
agg = collections.defaultdict(float); inst = collections.defaultdict(float); srcmap = {}
hdr = None
for x in r:
    if len(x) == 2 and x[0] == "File Path":
        cur_file = x[1].split("/")[-1]; continue
    if x and x[0] == "Line No":
        hdr = x; continue
    if hdr is None or len(x) < 8:
        continue
    if x[0]:
        cur_line, cur_src = x[0], x[1]
    try:
        v = float(x[4] or 0); ie = float(x[7] or 0)
    except ValueError:
        continue
    agg[(cur_file, cur_line)] += v; inst[(cur_file, cur_line)] += ie; srcmap[(cur_file, cur_line)] = cur_src
tot = sum(agg.values()); itot = sum(inst.values())
print(f"total samples {tot:.0f}, warp-instructions {itot:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v/tot*100:5.1f}% inst {inst[k]/itot*100:5.1f}%  {k[0]}:{k[1]}: {srcmap[k].strip()[:90]}")
