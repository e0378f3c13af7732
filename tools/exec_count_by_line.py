"""Executed warp instructions and stall samples per CUDA source line (ncu source page,
cuda+sass): where a kernel's issue slots go.  usage: exec_count_by_line.py REPORT [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, mode = None, None, None
ex = collections.Counter()
smp = collections.Counter()
src = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, isx = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].isdigit() or len(r) <= ie:
        continue
    key = (fname, int(r[0]))
    src.setdefault(key, r[1][:90])
    try:
        ex[key] += float(r[ie] or 0)
        smp[key] += float(r[isx] or 0)
    except ValueError:
        pass
tot, stot = sum(ex.values()), sum(smp.values())
print(f"executed warp instructions {tot:.0f}, stall samples {stot:.0f}")
for k, v in ex.most_common(top):
    print(f"{v:12.0f} {v / tot:6.3f} smp {smp[k] / max(stot, 1):6.3f}  {k[0]}:{k[1]}  {src[k].strip()}")
