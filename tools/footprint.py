"""Executed-code footprint of the fused kernel from an ncu report (source counters): SASS
instructions executed at least once (x 16 B), and the no_instruction share of the stall samples.
usage: footprint.py REPORT"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, n, ex = None, 0, 0
ranges = []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        n += 1
        try:
            e = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            e = 0
        if e > 0:
            ex += 1
print(f"sass {n} instructions ({n * 16 / 1024:.1f} KB), executed {ex} ({ex * 16 / 1024:.1f} KB)")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
tot = 0
st = {}
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st[k[33:]] = float(v[i])
        except ValueError:
            pass
tot = sum(st.values()) or 1
for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:6]:
    print(f"  stall {k}: {100 * x / tot:.1f}%")
for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum"):
    if k in h:
        print(" ", k, v[h.index(k)])
