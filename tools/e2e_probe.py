"""Where the host entry points spend a step (C4, 1M agents, exclusive context): host-timed
loops of the incremental path with and without the list read-back, the device step + sync
alone, and the empty-call floor.  Tools only."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2601_21473_b200.planner import Planner  # noqa: E402

n, S = 1_000_000, 40
w = bench.c4_shard(n, S, 1, 0)
b = w.blocks
pl = Planner(n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, transfer=False,
             device=0, keep_dist=False, exclusive=True)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
upd = [None]
for s in range(1, S):
    ch = np.nonzero(np.any(w.rec[s] != w.rec[s - 1], axis=1))[0].astype(np.uint32)
    upd.append((pin(ch), pin(w.rec[s][ch])))
pf = np.zeros(n, np.uint32)
ev = np.zeros(n, np.uint32)
rec0 = pin(w.rec[0])


def loop(kind):
    pl.step_host(int(w.now[0]), rec0, None, pf, ev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if kind == "submit":
        pl.submit_updates(int(w.now[1]), *upd[1])
        for s in range(1, S):
            if s + 1 < S:
                pl.submit_updates(int(w.now[s + 1]), *upd[s + 1])
            pl.collect(pf, ev)
        return (time.perf_counter() - t0) / (S - 1) * 1e6
    if kind in ("staged", "staged_nolists"):
        pl.stage_updates(*upd[1])
    for s in range(1, S):
        if kind == "staged" or kind == "staged_nolists":
            if s + 1 < S:
                pl.stage_updates(*upd[s + 1])
            if kind == "staged":
                pl.step_updates(int(w.now[s]), upd[s][0], upd[s][1], pf, ev)
            else:
                pl.step_updates(int(w.now[s]), upd[s][0], upd[s][1], None, None)
        elif kind == "unstaged":
            pl.step_updates(int(w.now[s]), upd[s][0], upd[s][1], pf, ev)
        elif kind == "device_step_sync":
            pl.step(int(w.now[s]))
            pl.sync()
        elif kind == "sync_only":
            pl.sync()
    return (time.perf_counter() - t0) / (S - 1) * 1e6


for rep in range(2):
    for kind in ("submit", "staged", "staged_nolists", "unstaged", "device_step_sync", "sync_only"):
        print(rep, kind, round(loop(kind), 1), "us/step", flush=True)
