"""Per-source-line warp-stall samples of an ncu report (CUDA source view): the lines with the
most samples and their dominant stall reasons.  Usage: ncu_lines.py REPORT [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, header = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] in ("Function Name", "Kernel Name"):
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header is None or not rec[0].isdigit():
        continue
    d = dict(zip(header, rec))
    try:
        n = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    rows.append((n, fname, int(rec[0]), d.get("Source", "").strip(), stalls, d.get("Instructions Executed", "")))
import os
src_cache = {}
def src_line(f, ln):
    if f not in src_cache:
        hits = [os.path.join(dp, f) for dp, _, fs in os.walk(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))) if f in fs]
        src_cache[f] = open(hits[0]).read().split("\n") if hits else []
    L = src_cache[f]
    return L[ln - 1].strip() if 0 < ln <= len(L) else ""
rows = [(n, f, ln, src if src not in ("", "-") else src_line(f, ln), st, ins) for n, f, ln, src, st, ins in rows]
tot = sum(r[0] for r in rows) or 1
print(f"total samples {tot}")
for n, f, ln, src, st, ins in sorted(rows, reverse=True)[:top]:
    s3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100*n/tot:5.1f}% {f}:{ln:<5} inst={ins:<9} {', '.join(f'{k[6:]}={v}' for k, v in s3):<55} {src[:90]}")
