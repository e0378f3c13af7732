"""Phase stamps of one C5 instance (10k agents, one CTA per instance) in a batched step of 148
instances: where a single-CTA plan spends its time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen as tg
from paper_2601_21473_b200.planner import Planner, step_batch

dev = torch.device("cuda", 0)
T = 12
n_inst = 148
traces = [tg.config_c5(replica=r, budget_pct=10 * (1 + r % 9), seed_base=100, steps=T) for r in range(16)]
recs = [torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(T, -1)).to(dev) for w in traces]
stream = torch.cuda.Stream(dev)
pls = []
for i in range(n_inst):
    w = traces[i % 16]
    b = w.blocks
    budget = int(w.footprint.sum()) * (10 * (1 + i % 9)) // 100
    pls.append(Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta, transfer=False,
                       device=0, stream=stream, keep_dist=False))
for s in range(T):
    for i, pl in enumerate(pls):
        pl.set_inputs_ptr(recs[i % 16][s].data_ptr())
    if s == T - 1:
        torch.cuda.synchronize()
        for pl in pls[:4]:
            pl.stamps(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_batch(pls, int(traces[0].now[s]))
    e1.record(stream)
    torch.cuda.synchronize()
    if s >= T - 3:
        print("step", s, "ms", round(e0.elapsed_time(e1), 4))
for j, pl in enumerate(pls[:4]):
    st = pl.stamps().astype(np.int64)
    r = lambda q: round((int(st[q]) - int(st[0])) / 1e3, 2) if st[q] else None
    h = pl.sync()
    print("inst", j, "npf", h["n_prefetch"], "nev", h["n_evict"], "| B1", r(4), "cleared", r(32), "coarse", r(33),
          "fine", r(34), "selbar", r(35), "sel", r(9), "P3", r(10), "| P1loop", r(25), "P1end", r(11), "P3end", r(14),
          "P4loop", r(27), "P4lists", r(17), "P4ranks", r(19), "P4rows", r(28), "P4end", r(12), "P5tables", r(13),
          "end", r(1), "| slots", int(st[16]), "slot_loop_ns", int(st[21]), "sections", [int(st[q]) for q in (22, 23, 24, 29)],
          "max_sorted_seg", int(st[18]))
