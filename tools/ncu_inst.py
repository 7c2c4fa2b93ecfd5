"""Per-source-line warp-instructions and stall samples from an ncu --set full report
(source rows only; SASS rows are not double counted).  Usage: ncu_inst.py REP [N]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = None
inst = collections.defaultdict(float); stall = collections.defaultdict(float); src = {}
for x in csv.reader(out.splitlines()):
    if len(x) == 2 and x[0] == "File Path":
        cur_file = x[1].split("/")[-1]; continue
    if not x or x[0] in ("Line No", "Function Name") or len(x) < 8 or not x[0]:
        continue
    try:
        k = (cur_file, int(x[0]))
        inst[k] += float(x[7] or 0); stall[k] += float(x[4] or 0); src[k] = x[1]
    except ValueError:
        continue
ti, ts = sum(inst.values()), sum(stall.values())
print(f"warp-instructions {ti:.4e}  stall samples {ts:.0f}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:n]:
    print(f"inst {v/ti*100:5.1f}%  stall {stall[k]/ts*100:5.1f}%  {k[0]}:{k[1]}: {src[k].strip()[:95]}")
