"""Warp-instructions and stall samples of ess_kernel per phase (source-line ranges of
ess_chain.cu; inlined helpers of common.cuh attributed by function).  Tooling."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
inst = collections.defaultdict(float); stall = collections.defaultdict(float)
for x in csv.reader(out.splitlines()):
    if len(x) == 2 and x[0] == "File Path":
        cur = x[1].split("/")[-1]; continue
    if not x or x[0] in ("Line No", "Function Name") or len(x) < 8 or not x[0]:
        continue
    try:
        k = (cur, int(x[0])); inst[k] += float(x[7] or 0); stall[k] += float(x[4] or 0)
    except ValueError:
        pass
ranges = [(int(a), int(b), n) for a, b, n in (r.split(":") for r in sys.argv[2].split(","))]
def phase(k):
    f, l = k
    if f == "common.cuh":
        if 90 <= l <= 140: return "rng (philox/box-muller)"
        if 170 <= l <= 245: return "nu digits"
        if 260 <= l <= 380: return "arcs (arc_of/atan2)"
        if 30 <= l <= 60: return "tiled offsets"
        return "common other"
    if f != "ess_chain.cu": return f
    for a, b, n in ranges:
        if a <= l <= b: return n
    return "ess other"
I = collections.defaultdict(float); Sx = collections.defaultdict(float)
for k in inst: I[phase(k)] += inst[k]; Sx[phase(k)] += stall[k]
ti, ts = sum(I.values()), sum(Sx.values())
print(f"total warp-instructions {ti:.4e}")
for n, v in sorted(I.items(), key=lambda kv: -kv[1]):
    print(f"{n:32s} inst {v/ti*100:5.1f}%  stall {Sx[n]/ts*100:5.1f}%")
