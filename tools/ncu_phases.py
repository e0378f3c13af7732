"""Warp-stall samples and executed instructions of an ncu report, aggregated by phase of
k_fused_plan (phase = the '---------------- Pn' marker comment preceding the source line).
Usage: ncu_phases.py REPORT [fused.cu]  (pass the source revision the report was built from)"""
import csv, io, subprocess, sys

rep = sys.argv[1]
srcf = sys.argv[2] if len(sys.argv) > 2 else "paper_2601_21473_b200/csrc/fused.cu"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, header = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header is None or not rec[0].isdigit():
        continue
    d = dict(zip(header, rec))
    try:
        n = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ins = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((str(fname), int(rec[0]), n, ins))
src = open(srcf).read().split("\n")
kstart = [i + 1 for i, l in enumerate(src) if "k_fused_plan(const" in l][0]
starts = [("prologue", kstart)]
for i, l in enumerate(src):
    if "// ----------------" in l and i + 1 > kstart:
        starts.append((l.split("----------------")[1].strip()[:24], i + 1))


def phase(ln):
    if ln < kstart:
        return "helpers in fused.cu"
    p = "prologue"
    for nm, s in starts:
        if ln >= s:
            p = nm
    return p


agg = {}
for f, ln, n, ins in rows:
    k = phase(ln) if f == "fused.cu" else "inlined from " + f
    a = agg.setdefault(k, [0, 0])
    a[0] += n
    a[1] += ins
tot = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
for k, (n, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:40s} samples {100 * n / tot:5.1f}%  warp-inst {ins:9d} ({100 * ins / ti:4.1f}%)")
print("total warp instructions", ti, "samples", tot)
