"""Export one kernel's raw metrics from an ncu report to JSON (profiles/), and refresh
profiles/latest_traffic.json (DRAM bytes per launch, read by bench.py's roofline.traffic).
Usage: export_ncu.py REPORT OUT_JSON [KERNEL_PREFIX]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
prefix = sys.argv[3] if len(sys.argv) > 3 else "k_fused_plan"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, data = rows[0], rows[1], rows[2:]
ki = hdr.index("Kernel Name")
sel = [r for r in data if prefix in r[ki]]
r = sel[-1]
d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
res = {h: v for h, (v, u) in d.items()}
res["_units"] = {h: u for h, (v, u) in d.items() if u}
json.dump(res, open(out, "w"), indent=0, sort_keys=True)


def num(k):
    return float(res[k].replace(",", ""))


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale.get(res["_units"].get("dram__bytes_read.sum", "byte"), 1)
wr *= scale.get(res["_units"].get("dram__bytes_write.sum", "byte"), 1)
print(json.dumps({"kernel": r[ki][:80], "dram_read": rd, "dram_write": wr,
                  "duration": res.get("gpu__time_duration.sum"), "unit": res["_units"].get("gpu__time_duration.sum")}))
json.dump({"kernel_prefix": prefix, "dram_bytes_per_launch": rd + wr, "source": out + " (ncu --set full, one steady-state launch, C4 1M agents)",
           "algorithmic_bytes_per_launch": 16250000.0}, open("profiles/latest_traffic.json", "w"), indent=1)
