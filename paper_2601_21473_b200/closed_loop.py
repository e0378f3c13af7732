"""Closed-loop step simulation (NEXT #3): a trace of agent records is planned step after step
under one of the three presets of the paper's evaluation (§4.1 baselines; SPEC
S:477-480 PresetName = (eviction, prefetch, prefix backing)):

  scalesim     (invocation distance, distance-guided prefetch, host-backed) — the planner as
               configured (alias "distance");
  hicache_like (LRU, no prefetch, host-backed: evicted dirty KV / history blocks are written
               back and reloaded, "SGLang's default hierarchical caching"; alias "lru");
  sglang_like  (LRU, no prefetch, no host backing: evicted KV / history blocks are dropped and
               recomputed on the next use, "radix-structured prefix cache without CPU
               fallback"; LoRA adapters are host-backed in every preset).

LRU is expressed as explicit distances (scalesim_lru_records, reading R20) and planned with
theta = 0.  Every planning step runs in the library's kernels; the per-step accounting here
reads the plan's outputs back.

Per step: demand misses (agents that need their memory now — distance 0 — and were not
resident before the step's plan: loads on the critical path), bytes loaded,
written back, recomputed; and stalls under a transfer-time model (reading R24): one host link
of `link_GBs`, loads issued at the start of their plan's step in list order (most urgent
first) on one channel, a step lasting `step_s`; an agent whose LLM call starts at step
r (phase WAITING) waits until its load completes: stall = max(0, completion - r * step_s).
Recompute (sglang_like) is not a transfer and is reported as bytes only.  With prefetch, the load of
an agent needed d steps ahead has d steps to finish ("the prefetch operation can proceed
in parallel"); a demand load waits for its whole transfer (SPEC acceptance #3).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .planner import Planner

PRESETS = {"scalesim": "scalesim", "distance": "scalesim", "hicache_like": "hicache_like", "lru": "hicache_like",
           "sglang_like": "sglang_like"}


def run(rec_steps, now_steps, blk_ptr, blk_size, blk_host_off, blk_kind, budget: int, theta, policy: str,
        hop_scale: float = 1.0, device: int = 0, multi_kernel: bool = False, link_GBs: float = 55.0,
        step_s: float = 1.0):
    """rec_steps: (T, n, 4) uint32 agent records; policy: a preset name (or "distance" /
    "lru").  Returns a dict of per-step arrays: misses, miss_bytes, loaded_bytes,
    writeback_bytes, recompute_bytes, stall_s, n_prefetch, n_evict."""
    preset = PRESETS[policy]
    rec_steps = np.ascontiguousarray(rec_steps, dtype=np.uint32)
    T, n = rec_steps.shape[0], rec_steps.shape[1]
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(dev)
    lru = preset != "scalesim"
    th = np.zeros(3, np.float32) if lru else np.asarray(theta, np.float32)
    pl = Planner(n, blk_ptr, blk_size, blk_host_off, blk_kind, budget, th, hop_scale=hop_scale, transfer=False,
                 device=device, stream=stream, keep_dist=True, multi_kernel=multi_kernel, explicit_dist=lru)
    lib = L.lib()
    agent_rec = torch.zeros(n * 16, dtype=torch.uint8, device=dev)
    last_use = torch.full((n,), -1, dtype=torch.int32, device=dev)  # 0xFFFFFFFF: never used
    out = {k: np.zeros(T, np.int64) for k in ("misses", "miss_bytes", "loaded_bytes", "writeback_bytes",
                                              "recompute_bytes", "n_prefetch", "n_evict")}
    out["stall_s"] = np.zeros(T, np.float64)
    fp = rec_steps[:, :, 1].astype(np.int64)
    # per-agent KV + history bytes (dropped and recomputed under sglang_like)
    bp = np.asarray(blk_ptr, np.int64)
    kvb = np.zeros(n, np.int64)
    kinds, sizes = np.asarray(blk_kind), np.asarray(blk_size, np.int64)
    nz = np.nonzero(np.diff(bp))[0]
    for a in nz:
        s = slice(int(bp[a]), int(bp[a + 1]))
        kvb[a] = int(sizes[s][kinds[s] != 0].sum())
    dropped = np.zeros(n, bool)   # sglang_like: KV / history gone since the last eviction
    ready_at = np.full(n, -np.inf)  # completion time of the agent's last load
    channel = 0.0                   # the host link's busy-until time
    bw = link_GBs * 1e9
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
        out["n_prefetch"][t] = hdr["n_prefetch"]
        out["n_evict"][t] = hdr["n_evict"]
        if preset == "sglang_like":
            # no host copy of KV / history: nothing is written back, the dropped part of a
            # reloaded agent is recomputed (not moved over the link)
            out["writeback_bytes"][t] = 0
            rec_pf = pf[dropped[pf]]
            out["recompute_bytes"][t] = int(kvb[rec_pf].sum())
            moved = fp[t, pf] - np.where(dropped[pf], kvb[pf], 0)
            out["loaded_bytes"][t] = int(moved.sum())
            dropped[pf] = False
            dropped[ev] = True
        else:
            out["writeback_bytes"][t] = hdr["bytes_d2h"]
            out["loaded_bytes"][t] = hdr["bytes_h2d"]
            moved = fp[t, pf]
        # the link: this step's loads in list order (most urgent first), after the previous ones
        t0 = t * step_s
        channel = max(channel, t0)
        done = channel + np.cumsum(moved) / bw
        if len(pf):
            channel = float(done[-1])
            ready_at[pf] = done
        ready_at[ev] = -np.inf
        need = np.nonzero((rec_steps[t][:, 2] & 3) == 1)[0]  # LLM calls starting now (WAITING)
        out["stall_s"][t] = float(np.maximum(0.0, ready_at[need] - t0).sum())
    pl.close()
    return out
