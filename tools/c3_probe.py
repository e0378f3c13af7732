"""C3 planning only (100k agents, three classes): a few steps of score + plan, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen as tg
from paper_2601_21473_b200.planner import Planner

w = tg.config_c3(seed=1, steps=6)
b = w.blocks
pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, hop_scale=w.hop_scale,
             n_kin=w.n_kin, page_bytes=w.page_bytes, transfer=False, keep_dist=False)
for s in range(w.steps):
    pl.set_records(w.rec[s], w.kin[s])
    pl.step(int(w.now[s]))
    h = pl.sync()
    print(s, h["n_prefetch"], h["n_evict"], h["status"], flush=True)
acting_int = ((w.rec[-1][:, 2] & 3) == 0) & (((w.rec[-1][:, 2] >> 2) & 3) == 1)
print("acting interaction agents", int(acting_int.sum()))
