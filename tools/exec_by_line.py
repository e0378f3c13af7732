"""Executed SASS instructions per CUDA source line (ncu source page, cuda+sass): where the
kernel's executed code footprint comes from.  usage: exec_by_line.py REPORT [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, hdr = None, None, None
cnt = collections.Counter()
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        line = (fname, int(r[0])) if r[0].isdigit() else None
        continue
    if line and len(r) > 7:
        try:
            if int(r[7] or 0) > 0:
                cnt[line] += 1
        except ValueError:
            pass
tot = sum(cnt.values())
print("executed SASS instructions", tot)
by_range = collections.Counter()
for (f, ln), n in cnt.items():
    by_range[(f, ln // 25 * 25)] += n
for (f, ln), n in sorted(by_range.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{n:5d}  {f}:{ln}-{ln + 24}")
