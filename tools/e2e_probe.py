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
    if kind == "submit_empty":  # the same loop with no changed records (no H2D, no scatter work)
        e = (pin(np.zeros(0, np.uint32)), pin(np.zeros((0, 4), np.uint32)))
        pl.submit_updates(int(w.now[1]), *e)
        pl.submit_updates(int(w.now[2]), *e)
        for s in range(1, S):
            if s + 2 < S:
                pl.submit_updates(int(w.now[s + 2]), *e)
            pl.collect(pf, ev)
        return (time.perf_counter() - t0) / (S - 1) * 1e6
    if kind == "h2d_only":  # the updates' copies alone on a side stream, back to back
        st = torch.cuda.Stream()
        dst = torch.empty(20 * n, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            for s in range(1, S):
                dst[:upd[s][0].nbytes].copy_(torch.from_numpy(upd[s][0].view(np.uint8)), non_blocking=True)
                dst[upd[s][0].nbytes:upd[s][0].nbytes + upd[s][1].nbytes].copy_(
                    torch.from_numpy(upd[s][1].view(np.uint8).reshape(-1)), non_blocking=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / (S - 1) * 1e6
    if kind == "submit":
        pl.submit_updates(int(w.now[1]), *upd[1])
        pl.submit_updates(int(w.now[2]), *upd[2])
        ts = tc = 0.0
        for s in range(1, S):
            if s + 2 < S:
                a = time.perf_counter()
                pl.submit_updates(int(w.now[s + 2]), *upd[s + 2])
                ts += time.perf_counter() - a
            a = time.perf_counter()
            pl.collect(pf, ev)
            tc += time.perf_counter() - a
        print("   submit call", round(ts / (S - 3) * 1e6, 1), "us, collect call", round(tc / (S - 1) * 1e6, 1), "us")
        return (time.perf_counter() - t0) / (S - 1) * 1e6
    if kind == "enqueue_only":  # host cost of pl.step while the GPU is blocked by a spin kernel
        with torch.cuda.stream(pl.stream):
            torch.cuda._sleep(int(2e9 * 0.02))
        t0 = time.perf_counter()
        for s in range(1, S):
            pl.step(int(w.now[s]))
        el = (time.perf_counter() - t0) / (S - 1) * 1e6
        pl.sync()
        return el
    if kind == "enqueue_submit":  # host cost of submit_updates alone (GPU blocked, both slots)
        with torch.cuda.stream(pl.stream):
            torch.cuda._sleep(int(2e9 * 0.02))
        t0 = time.perf_counter()
        pl.submit_updates(int(w.now[1]), *upd[1])
        pl.submit_updates(int(w.now[2]), *upd[2])
        el = (time.perf_counter() - t0) / 2 * 1e6
        pl.collect(pf, ev)
        pl.collect(pf, ev)
        return el
    if kind in ("collect_ready", "collect_ready_nolists"):  # host cost of collect on a finished step
        tc = 0.0
        for s in range(1, 31, 3):
            for j in range(3):
                pl.submit_updates(int(w.now[s + j]), *upd[s + j])
            torch.cuda.synchronize()
            time.sleep(0.002)
            for j in range(3):
                a = time.perf_counter()
                if kind == "collect_ready":
                    pl.collect(pf, ev)
                else:
                    pl.collect(None, None)
                tc += time.perf_counter() - a
        return tc / 30 * 1e6
    if kind == "device_loop":  # device path only, same records resident: K steps enqueued, one sync
        for s in range(1, S):
            pl.step(int(w.now[s]))
        pl.sync()
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
    for kind in ("enqueue_only", "enqueue_submit", "collect_ready", "collect_ready_nolists", "submit_empty", "h2d_only", "submit", "device_loop", "staged", "staged_nolists", "unstaged", "device_step_sync", "sync_only"):
        print(rep, kind, round(loop(kind), 1), "us/step", flush=True)
