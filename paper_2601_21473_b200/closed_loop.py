"""Closed-loop step simulation (NEXT #3): a trace of agent records is planned step after step
by the invocation-distance policy (the planner as configured) or by the reactive LRU baseline
of the paper's evaluation (on-demand loads, least-recently-used eviction; expressed as
explicit distances by scalesim_lru_records, reading R20, and planned with theta = 0).

Per step it reports the demand misses — agents that need their memory now (distance 0) and
were not resident before the step's plan, i.e. loads on the critical path —
and the bytes loaded and written back.  Every planning step runs in the library's kernels; the
per-step counting here reads the plan's outputs back.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .planner import Planner


def run(rec_steps, now_steps, blk_ptr, blk_size, blk_host_off, blk_kind, budget: int, theta, policy: str,
        hop_scale: float = 1.0, device: int = 0, multi_kernel: bool = False):
    """rec_steps: (T, n, 4) uint32 agent records; policy "distance" or "lru".  Returns a dict
    of per-step arrays: misses, miss_bytes, loaded_bytes, writeback_bytes, n_prefetch, n_evict."""
    assert policy in ("distance", "lru")
    rec_steps = np.ascontiguousarray(rec_steps, dtype=np.uint32)
    T, n = rec_steps.shape[0], rec_steps.shape[1]
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)
    lru = policy == "lru"
    th = np.zeros(3, np.float32) if lru else np.asarray(theta, np.float32)
    pl = Planner(n, blk_ptr, blk_size, blk_host_off, blk_kind, budget, th, hop_scale=hop_scale, transfer=False,
                 device=device, stream=stream, keep_dist=True, multi_kernel=multi_kernel, explicit_dist=lru)
    lib = L.lib()
    agent_rec = torch.zeros(n * 16, dtype=torch.uint8, device=dev)
    last_use = torch.full((n,), -1, dtype=torch.int32, device=dev)  # 0xFFFFFFFF: never used
    out = {k: np.zeros(T, np.int64) for k in ("misses", "miss_bytes", "loaded_bytes", "writeback_bytes",
                                              "n_prefetch", "n_evict")}
    fp = rec_steps[:, :, 1].astype(np.int64)
    for t in range(T):
        if lru:
            with torch.cuda.stream(stream):
                agent_rec.copy_(torch.from_numpy(rec_steps[t].view(np.uint8).reshape(-1)), non_blocking=False)
            L.check(lib.scalesim_lru_records(agent_rec.data_ptr(), n, int(now_steps[t]), last_use.data_ptr(),
                                             pl.rec.data_ptr(), stream.cuda_stream), "scalesim_lru_records")
        else:
            pl.set_records(rec_steps[t])
        pl.step(int(now_steps[t]))
        hdr = pl.sync()
        pf, ev = pl.lists(hdr)
        d = pl.distances()
        demand = pf[d[pf] == 0.0]  # needed now, not resident before the plan
        out["misses"][t] = len(demand)
        out["miss_bytes"][t] = int(fp[t, demand].sum())
        out["loaded_bytes"][t] = hdr["bytes_h2d"]
        out["writeback_bytes"][t] = hdr["bytes_d2h"]
        out["n_prefetch"][t] = hdr["n_prefetch"]
        out["n_evict"][t] = hdr["n_evict"]
    pl.close()
    return out
