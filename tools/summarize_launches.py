"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel rows."""
import collections
import csv
import json
import sys


def summarize(path, steps=None):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) <= max(ki, vi, ui):
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
                    "share": sum(v) / tot})
    return {"total_us": tot, "kernels": out}


if __name__ == "__main__":
    s = summarize(sys.argv[1])
    if len(sys.argv) > 2:
        json.dump(s, open(sys.argv[2], "w"), indent=1)
    for r in s["kernels"]:
        print(f"{r['kernel']:40s} n={r['launches']:4d} mean={r['mean_us']:9.2f}us share={r['share']:.3f}")
