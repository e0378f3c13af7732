"""One-off probe of the GPU box: host cores, RAM, GPU, pinned host<->device bandwidth."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception as e:
    out["cpu_model"] = str(e)
out["meminfo"] = open("/proc/meminfo").readline().strip()
out["gpu"] = torch.cuda.get_device_name(0)
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["mem_gb"] = p.total_memory / 1e9
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
def bw(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best
out["h2d_GBs"] = n / bw(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBs"] = n / bw(lambda: h.copy_(d, non_blocking=True)) / 1e9
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("topo", "smi")}))
