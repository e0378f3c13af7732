#!/usr/bin/env python
"""Benchmark of the ScaleSim planner hot path (BASELINE.json metric):
  agent-plans/sec (1M agents per GPU, 1/2/4/8 B200) and % HBM roofline; transfer GB/s vs
  the host link measured in the same run.

One step = score + plan (+ transfer call, a no-op for logical sizes) of every agent of the
C4 workload (1M independent AgentSociety-shaped agents per GPU, budget 25% of agent memory,
theta = 4, logical block sizes).  Inputs are resident in HBM; every timed step reads its own
16 MB record buffer (K distinct buffers, > 126 MB L2), so no step is served from L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

For N > 1 launch with torchrun (one rank per GPU); agents shard by contiguous id, the global
budget cut runs over NCCL inside the library (weak scaling: 1M agents per GPU).
`--impl reference` times the CPU oracle (the reference arm of this tier) on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tracegen as tg  # noqa: E402

WARM_IN = 16  # untimed trace steps that bring residency to steady state before warmup
BYTES_PER_AGENT_SCORE = 16.125  # k_score algorithmic bytes: 16 B record + 1/8 B residency bit
BYTES_PER_AGENT_STEP = 16.25  # whole step: record + old and new residency bits


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML in a thread during the timed region."""

    def __init__(self, dev=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def sample(self):
        N = self.N
        if N is None:
            return
        if not hasattr(self, "_names"):
            self._names = {getattr(N, k): k for k in dir(N) if k.startswith("nvmlClocksEventReason") or
                           k.startswith("nvmlClocksThrottleReason")}
        try:
            self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                N, "nvmlDeviceGetCurrentClocksEventReasons") else N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            for bit, name in self._names.items():
                if isinstance(bit, int) and bit and (r & bit) == bit and bit & (bit - 1) == 0:
                    self.reasons.add(name.replace("nvmlClocksEventReason", "").replace(
                        "nvmlClocksThrottleReason", ""))
        except Exception:
            pass

    def poll_until(self, event):
        """Sample from the calling thread until `event` (recorded at the end of the timed
        region) completes: the host enqueues ahead, so the GPU is still in the region."""
        while not event.query():
            self.sample()
            time.sleep(0.0005)

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N:
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"None", "GpuIdle", "ApplicationsClocksSetting"}),
                "samples": len(self.samples)}


def c4_shard(n_local: int, steps: int, seed: int, rank: int):
    """The C4 trace of this rank's shard (independent agents, C3 footprints, logical sizes)."""
    w = tg.config_c4(seed=seed + 1000 * rank, steps=steps, n=n_local)
    return w


def oracle_steps(w, steps, res=None, budget=None):
    import oracle
    res = np.zeros(w.n, np.uint8) if res is None else res
    budget = w.budget if budget is None else budget
    for s in steps:
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        p = oracle.plan(w.rec[s], d, res, w.theta, budget)
        res = p["resident"]
    return res


def cpu_baseline(w, target_s=10.0, max_s=30.0):
    """The oracle as it stands, single-threaded, on a bounded sample of the same workload."""
    import oracle
    res = oracle_steps(w, range(min(WARM_IN, w.steps)))
    t0 = time.perf_counter()
    n_steps = 0
    s = WARM_IN
    while True:
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        res = p["resident"]
        n_steps += 1
        s = s + 1 if s + 1 < w.steps else WARM_IN
        el = time.perf_counter() - t0
        if el >= target_s or el >= max_s:
            break
    return {"value": w.n * n_steps / el, "unit": "agent-plans/s", "cores": 1, "kind": "oracle",
            "sample": f"C4 shard of {w.n} agents, {n_steps} consecutive steps after a {WARM_IN}-step warm-in, "
                      f"score+plan, single thread, {el:.1f} s"}


def run_reference(args, rank, world):
    """Reference arm of this tier: the CPU oracle on the same workload (rank 0 only)."""
    if rank != 0:
        return
    n = args.n
    w = c4_shard(n, WARM_IN + args.warmup + args.steps, args.seed, 0)
    res = oracle_steps(w, range(WARM_IN + args.warmup))
    import oracle
    t0 = time.perf_counter()
    for s in range(WARM_IN + args.warmup, WARM_IN + args.warmup + args.steps):
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        res = p["resident"]
    el = time.perf_counter() - t0
    v = n * args.steps / el
    line = {"metric": "agent-plans/sec (1M agents, 1/2/4/8 B200) % HBM roofline; transfer GB/s vs host link",
            "impl": "reference", "value": v, "unit": "agent-plans/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"c4: {n} independent agents (AgentSociety-shaped), budget 25%, theta 4, "
                                   "logical sizes", "n_agents": n},
            "cpu_baseline": {"value": v, "unit": "agent-plans/s", "cores": 1, "kind": "oracle",
                             "sample": f"full workload, {args.steps} steps after {WARM_IN + args.warmup} warm steps"},
            "e2e": {"value": v, "unit": "agent-plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def link_peak(torch, dev):
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def best(fn, reps=6):
        b = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            b = min(b, time.perf_counter() - t)
        return b

    def bidir():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    r = {"h2d_GBs": n / best(lambda: d.copy_(h, non_blocking=True)) / 1e9,
         "d2h_GBs": n / best(lambda: h.copy_(d, non_blocking=True)) / 1e9,
         "bidir_GBs": 2 * n / best(bidir) / 1e9}
    del h, d, h2, d2
    return r


def transfer_leg(torch, dev, seed):
    """C2 (10k agents, 7B LoRA + KV pages, budget 25%): physical block transfers, timed
    with CUDA events on the copy stream; against the link peak measured here."""
    from paper_2601_21473_b200.planner import Planner
    w = tg.config_c2(seed=seed, steps=24, host_bytes=8 << 30)
    b = w.blocks
    host = torch.empty(int(b.host_bytes), dtype=torch.uint8, pin_memory=True)
    pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                 page_bytes=w.page_bytes, transfer=True, host_arena=host, device=dev.index)
    tot_b, tot_t, steps = 0, 0.0, 0
    h2d_b = d2h_b = 0
    for s in range(w.steps):
        pl.set_records(w.rec[s])
        pl.score(int(w.now[s]))
        pl.plan()
        pl.stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pl.copy_stream)
        pl.transfer()
        e1.record(pl.copy_stream)
        hdr = pl.sync()
        if s >= 8:  # steady state
            moved = hdr["n_h2d"] * w.page_bytes + hdr["n_d2h"] * w.page_bytes
            tot_b += moved
            h2d_b += hdr["n_h2d"] * w.page_bytes
            d2h_b += hdr["n_d2h"] * w.page_bytes
            tot_t += e0.elapsed_time(e1) / 1e3
            steps += 1
    pl.close()
    del host
    return {"bytes_per_step": tot_b / max(steps, 1), "h2d_bytes_per_step": h2d_b / max(steps, 1),
            "d2h_bytes_per_step": d2h_b / max(steps, 1), "GBs": tot_b / max(tot_t, 1e-12) / 1e9,
            "steps": steps, "workload": "c2: 10k agents, 7B rank-16 LoRA + 917,504 B KV pages, budget 25%, "
                                        "host arena 8 GiB (offsets aliased), TMA bulk page copies (2 x 8 CTAs)"}


def c3_leg(torch, dev, seed=1, warm=4, steps=8):
    """C3 (BASELINE configs[2]: 100k agents of all three classes, 80 GB budget, Qwen2.5-0.5B
    sizes): planning (with the interaction pair scan on the spatial grid) and physical
    transfers, then the same steps with each step's transfer overlapped with the next step's
    planning.  overlap efficiency = (t_plan + t_transfer) / t_overlapped."""
    from paper_2601_21473_b200.planner import Planner
    T = warm + steps
    w = tg.config_c3(seed=seed, steps=T, host_bytes=8 << 30)
    b = w.blocks
    recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(T, -1)).to(dev)
    kins = torch.from_numpy(np.ascontiguousarray(w.kin).view(np.uint8).reshape(T, -1)).to(dev)

    def mk(transfer, host=None):
        return Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                       hop_scale=w.hop_scale, n_kin=w.n_kin, page_bytes=w.page_bytes, transfer=transfer,
                       host_arena=host, device=dev.index, keep_dist=False)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # (1) planning alone (score = the a1' pair scan + deferral; plan = the fused kernel)
    pl = mk(False)
    t_score, t_plan = [], []
    for s in range(T):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        e = [ev() for _ in range(3)]
        e[0].record(pl.stream)
        pl.score(int(w.now[s]))
        e[1].record(pl.stream)
        pl.plan()
        e[2].record(pl.stream)
        torch.cuda.synchronize(dev)
        if s >= warm:
            t_score.append(e[0].elapsed_time(e[1]))
            t_plan.append(e[0].elapsed_time(e[2]))
    pl.close()
    host = torch.empty(int(b.host_bytes), dtype=torch.uint8, pin_memory=True)
    # (2) the same steps, each transfer timed alone (plan, wait, transfer, wait)
    pl = mk(True, host)
    t_x, moved = [], []
    for s in range(T):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        pl.score(int(w.now[s]))
        pl.plan()
        pl.stream.synchronize()
        e0, e1 = ev(), ev()
        e0.record(pl.copy_stream)
        pl.transfer()
        e1.record(pl.copy_stream)
        hdr = pl.sync()
        if s >= warm:
            t_x.append(e0.elapsed_time(e1))
            moved.append((hdr["n_h2d"] + hdr["n_d2h"]) * w.page_bytes)
    pl.close()
    torch.cuda.empty_cache()
    # (3) the same steps back to back: transfer t runs on the copy streams while plan t+1 runs
    # on the planner stream; events bracket every plan (planner stream) and every transfer
    # (copy stream), so the overlap is read off the device timeline directly
    pl = mk(True, host)
    for s in range(warm):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        pl.step(int(w.now[s]))
    pl.sync()
    e0, e1 = ev(), ev()
    pa = [ev() for _ in range(steps)]
    pb = [ev() for _ in range(steps)]
    xe = [ev() for _ in range(steps)]
    with torch.cuda.stream(pl.stream):
        torch.cuda._sleep(int(1e8))
    e0.record(pl.stream)
    for k, s in enumerate(range(warm, T)):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        pa[k].record(pl.stream)
        pl.score(int(w.now[s]))
        pl.plan()
        pb[k].record(pl.stream)
        pl.transfer()
        xe[k].record(pl.copy_stream)
    pl.join()
    e1.record(pl.stream)
    torch.cuda.synchronize(dev)
    t_over = e0.elapsed_time(e1) / steps
    # hidden share of plan k+1: the part of [start, end] of its plan that lies before the end
    # of transfer k (device timestamps relative to e0)
    hid = []
    for k in range(steps - 1):
        a, b, x = e0.elapsed_time(pa[k + 1]), e0.elapsed_time(pb[k + 1]), e0.elapsed_time(xe[k])
        hid.append(max(0.0, min(b, x) - a) / max(b - a, 1e-9))
    plan_in_overlap = float(np.mean([e0.elapsed_time(pb[k + 1]) - e0.elapsed_time(pa[k + 1]) for k in range(steps - 1)]))
    pl.close()
    del host
    torch.cuda.empty_cache()
    tp, tx = float(np.mean(t_plan)), float(np.mean(t_x))
    return {"workload": f"c3: {w.n} agents (independent / interaction / diffusion thirds), 80 GB budget, "
                        "0.5B LoRA + KV pages + history, host arena 8 GiB (offsets aliased)",
            "plan_ms": tp, "score_ms": float(np.mean(t_score)), "transfer_ms": tx,
            "bytes_per_step": float(np.mean(moved)), "transfer_GBs": float(np.mean(moved)) / (tx / 1e3) / 1e9,
            "step_ms_overlapped": t_over,
            "hidden_fraction": float(np.mean(hid)),
            "hidden_fraction_definition": "share of plan t+1's device interval (planner-stream events) that lies before "
                                          "the end of transfer t (copy-stream event), mean over steps",
            "planner_stream_interval_ms": plan_in_overlap,
            "planner_stream_note": "per step, the planner stream's interval from the step's score to the end of its plan; it "
                                   "includes waiting for the descriptor buffer of step t-2 (two plans ahead of the copies), "
                                   "not plan work (the plan kernels alone: plan_ms)",
            "copy_sms": "2 launches x 8 CTAs (write-backs | independent loads); the plan kernel runs on the other 132 SMs",
            "hidden_fraction_formula": (tp + tx - t_over) / tp,
            "hidden_fraction_formula_note": "(t_plan + t_transfer - t_overlapped) / t_plan from separately timed runs: "
                                            "differences of ~265 ms transfer times, noise-dominated at t_plan ~0.2 ms",
            "value": w.n / (t_over / 1e3), "unit": "agent-plans/s (planning + transfer, overlapped)",
            "steps": steps}


def closed_loop_leg(dev, steps=64, seed=1):
    """NEXT #3: C2 (10k agents, 7B LoRA + KV pages, budget 25%) stepped in closed loop under the
    three presets of the paper's evaluation: scalesim (invocation distance,
    prefetch), hicache_like (LRU, host-backed) and sglang_like (LRU, KV dropped and recomputed),
    with stalls under the transfer-time model (55 GB/s link, 1 s per simulation step); and the scalesim
    preset on estimated action ends (S:187 noise knob, sigma 0.5)."""
    from paper_2601_21473_b200 import closed_loop
    res = {}
    warm = 8  # the first steps fill the empty GPU under every preset
    for name, pol, noise in (("scalesim", "scalesim", 0.0), ("hicache_like", "hicache_like", 0.0),
                             ("sglang_like", "sglang_like", 0.0), ("scalesim_noise0.5", "scalesim", 0.5)):
        w = tg.config_c2(seed=seed, steps=steps, noise=noise)
        b = w.blocks
        o = closed_loop.run(w.rec, w.now, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                            policy=pol, device=dev.index)
        res[name] = {"demand_misses": int(o["misses"][warm:].sum()), "demand_miss_GB": float(o["miss_bytes"][warm:].sum()) / 1e9,
                     "loaded_GB": float(o["loaded_bytes"][warm:].sum()) / 1e9,
                     "written_back_GB": float(o["writeback_bytes"][warm:].sum()) / 1e9,
                     "recomputed_GB": float(o["recompute_bytes"][warm:].sum()) / 1e9,
                     "stall_s": float(o["stall_s"][warm:].sum())}
    d, l = res["scalesim"], res["hicache_like"]
    return {"workload": f"c2 closed loop: 10000 agents, {steps} steps (first {warm} excluded), budget 25%, theta 4",
            "presets": res,
            "demand_miss_reduction_vs_hicache": 1.0 - d["demand_misses"] / max(l["demand_misses"], 1),
            "stall_reduction_vs_hicache": 1.0 - d["stall_s"] / max(l["stall_s"], 1e-12),
            "note": "demand miss = an agent needed now (distance 0) that was not resident before the step's plan: "
                    "a load on the critical path (P:87, P:373-375); stall = time such an agent waits for its load "
                    "on one 55 GB/s channel, counted when its LLM call starts (reading R24)"}


def sweep_leg(torch, dev, peak_gbs, ns_m=(1, 2, 4, 8, 16, 32, 64), K=10, reps=5, seed=1):
    """N-sweep (SURVEY 8(d) "Report an N-sweep (1M..64M)"): the C4 population (1M independent
    AgentSociety-shaped agents, C3 footprints, budget 25%) replicated m times = m x 1M agents on
    one GPU, planned with the default kernel for its size (shared-memory tile up to 1.8M agents,
    the streaming variant above); per N: K eager steps per repeat, 5 repeats (median, p10,
    p90 of ms/step), each step reading its own record buffer; achieved HBM GB/s of the
    algorithmic 16.25 B/agent against the measured peak and the 8 TB/s datasheet figure."""
    from paper_2601_21473_b200.planner import Planner
    T1 = 6 + K
    w1 = tg.config_c4(seed=seed, steps=T1, n=1_000_000)
    fp1 = np.ascontiguousarray(w1.rec[0][:, 1]).astype(np.uint32)
    base = [torch.from_numpy(np.ascontiguousarray(w1.rec[s]).view(np.uint8).reshape(-1, 16)).to(dev) for s in range(T1)]
    out = []
    for m in ns_m:
        n = m * 1_000_000
        blk_ptr = np.arange(n + 1, dtype=np.uint64)
        blk_size = np.tile(fp1, m)
        pl = Planner(n, blk_ptr, blk_size, np.zeros(n, np.uint64), np.full(n, tg.KIND_KV, np.uint8), m * w1.budget,
                     w1.theta, transfer=False, device=dev.index, keep_dist=False, exclusive=True)
        del blk_ptr, blk_size
        recs = [b.repeat(m, 1).reshape(-1) for b in base]
        for s in range(6):
            pl.set_inputs_ptr(recs[s].data_ptr())
            pl.step(int(w1.now[s]))
        hdr = pl.sync()
        ms = []
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(pl.stream):
                torch.cuda._sleep(int(2e9 * 0.02 + K * 2e5 * max(1, m // 4)))
            e0.record(pl.stream)
            for k in range(K):  # (the same K record buffers each repeat; > L2 from 8M agents)
                s = 6 + k
                pl.set_inputs_ptr(recs[s].data_ptr())
                pl.step(int(w1.now[s]))
            e1.record(pl.stream)
            torch.cuda.synchronize(dev)
            ms.append(e0.elapsed_time(e1) / K)
        hdr = pl.sync()
        med = float(np.median(ms))
        gbs = n * BYTES_PER_AGENT_STEP / (med / 1e3) / 1e9
        out.append({"n_agents": n, "kernel": "streaming (fused_big)" if pl.big else ("shared-memory tile" if pl.fused else "multi-kernel"),
                    "ms_per_step_median": med, "ms_p10": float(np.percentile(ms, 10)), "ms_p90": float(np.percentile(ms, 90)),
                    "agent_plans_per_s": n / (med / 1e3), "hbm_GBs": gbs, "frac_measured_peak": gbs / peak_gbs,
                    "frac_8TBs": gbs / 8000.0, "status": hdr["status"], "n_prefetch": hdr["n_prefetch"]})
        pl.close()
        del recs
        torch.cuda.empty_cache()
    return {"workload": "C4 population replicated: m x (1M independent agents, C3 footprints, budget 25%, theta 4)",
            "repeats": reps, "steps_per_repeat": K, "launch_mode": "SCALESIM_F_EXCLUSIVE", "points": out}


def sched_leg(torch, dev, link=None, seed=3):
    """NEXT #2: the preemptive load scheduler (scalesim_sched_run) moving C2-sized agents
    (7B rank-16 LoRA + KV pages, ~24 MB each) in 16 MB chunks over the host link: 160 prefetch
    tasks at distances 1..12 submitted at slot 0, an urgent (distance 0) task every 6 slots,
    distance refreshes that cancel 10% of the waiting tasks; device-timed."""
    from paper_2601_21473_b200.planner import LOAD_EVENT, sched_run
    rng = np.random.default_rng(seed)
    n_agents, chunk = 256, 16 << 20
    per = 20_185_088 + 917_504 * 3
    host_bytes = 2 << 30
    host = torch.empty(host_bytes, dtype=torch.uint8, pin_memory=True)
    devm = torch.empty(n_agents * per, dtype=torch.uint8, device=dev)
    evs = []
    for a in range(160):
        evs.append((0, 0, a, float(rng.integers(1, 13)), (a * per) % (host_bytes - per) // 16 * 16, a * per, per))
    for k, a in enumerate(range(160, 256)):
        # (odd slots: the urgent task lands between the two chunks of a running prefetch)
        evs.append((6 * (k + 1) + 1, 0, a, 0.0, (a * per) % (host_bytes - per) // 16 * 16, a * per, per))
        if k % 2 == 0:
            b = int(rng.integers(0, 160))
            evs.append((6 * (k + 1) + 1, 1, b, 20.0, 0, 0, 0))
    evs.sort(key=lambda e: e[0])
    ev = np.array(evs, dtype=LOAD_EVENT)
    sched_run(ev[:4], n_agents, 12.0, chunk, host, devm, 100_000)  # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream(dev)
    e0.record(st)
    out = sched_run(ev, n_agents, 12.0, chunk, host, devm, 100_000, sync=False)
    e1.record(st)
    torch.cuda.synchronize(dev)
    trace_t, tasks_t, counts_t = out[0], out[1], out[2]
    c = counts_t.cpu().numpy().view(np.uint32)
    tr = trace_t.cpu().numpy().view(np.uint32).reshape(-1, 2)[:c[0]]
    tk = tasks_t.cpu().numpy()[:c[1] * 32].view(np.dtype([("agent", "<u4"), ("chunks", "<u4"), ("done", "<u4"),
                                                          ("state", "<u4"), ("priority", "<f4"),
                                                          ("preemptions", "<u4"), ("finish_slot", "<u4"), ("pad", "<u4")]))
    moved = 0
    for t, k in tr:
        if t != 0xFFFFFFFF:
            moved += min(chunk, per - int(k) * chunk)
    ms = e0.elapsed_time(e1)
    urgent = tk[tk["priority"] == 0.0]
    wait = [int(u["finish_slot"]) for u in urgent]
    r = {"workload": "C2-sized agents (20.2 MB LoRA + 3 KV pages), 160 prefetch tasks at distances 1..12 at slot 0, "
                     "an urgent distance-0 task every 6 slots (96, landing mid-task: preemptions), distance refreshes cancelling "
                     "waiting tasks",
         "chunk_bytes": chunk, "slots": int(c[0]), "tasks": int(c[1]), "bytes_moved": moved, "ms": ms,
         "GBs": moved / (ms / 1e3) / 1e9, "preemptions": int(tk["preemptions"].sum()),
         "cancelled": int((tk["state"] == 4).sum()), "done": int((tk["state"] == 3).sum()),
         "urgent_tasks": int(len(urgent))}
    if link:
        r["frac_of_h2d_link"] = r["GBs"] / link["h2d_GBs"]
    del host, devm
    return r


def c5_leg(torch, dev, rank, world, replicas=64, budgets=tuple(range(10, 100, 10)), steps=8, warm=8, seed_base=100):
    """C5: independent simulation replicas x budget sizes, instances sharded over the ranks
    (instance i on rank i % world), all of a rank's instances stepped by scalesim_step_batch.
    Returns this rank's agent-plans and the device time of the timed steps."""
    from paper_2601_21473_b200.planner import Planner, step_batch
    T = warm + steps
    mine = [(r, pct) for i, (r, pct) in enumerate((r, p) for r in range(replicas) for p in budgets) if i % world == rank]
    reps = sorted({r for r, _ in mine})
    traces = {r: tg.config_c5(replica=r, budget_pct=10, seed_base=seed_base, steps=T) for r in reps}
    recs = {r: torch.from_numpy(np.ascontiguousarray(traces[r].rec).view(np.uint8).reshape(T, -1)).to(dev) for r in reps}
    stream = torch.cuda.Stream(dev)
    pls = []
    for r, pct in mine:
        w = traces[r]
        b = w.blocks
        budget = int(w.footprint.sum()) * pct // 100
        pls.append((r, Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta,
                               transfer=False, device=dev.index, stream=stream, keep_dist=False)))

    def one(s):
        for r, pl in pls:
            pl.set_inputs_ptr(recs[r][s].data_ptr())
        step_batch([pl for _, pl in pls], int(traces[reps[0]].now[s]))

    for s in range(warm):
        one(s)
    torch.cuda.synchronize(dev)
    lc0 = sum(pl.launch_count() for _, pl in pls)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e8))
    e0.record(stream)
    for s in range(warm, T):
        one(s)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    launches = sum(pl.launch_count() for _, pl in pls) - lc0
    n_agents = sum(traces[r].n for r, _ in pls)
    for _, pl in pls:
        pl.close()
    return {"instances": len(pls), "agents_per_step": n_agents, "steps": steps, "ms": ms,
            "launches": launches}


def objects_leg(torch, dev, n=1_000_000, steps=8, warm=8, seed=5):
    """NEXT #1: 1M C4 agents + shared memory objects (a system prompt shared by
    all, n/100 persona adapters, private KV pages): per step the agent plan (distances kept),
    scalesim_object_min, and the object plan (explicit distances), all on one stream."""
    from paper_2601_21473_b200.planner import Planner, object_min
    T = warm + steps
    w = tg.config_c4(seed=seed, steps=T, n=n)
    ob = tg.gen_objects(n, seed=seed)
    recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(T, -1)).to(dev)
    flags = torch.from_numpy(np.stack([ob.flags(w.rec[s]) for s in range(T)])).to(dev)
    stream = torch.cuda.Stream(dev)
    b = w.blocks
    agents = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, transfer=False,
                     device=dev.index, stream=stream, keep_dist=True)
    bo = ob.blocks
    ob_budget = int(ob.obj_bytes.astype(np.int64).sum()) // 4
    objs = Planner(ob.n, bo.blk_ptr, bo.blk_size, bo.blk_host_off, bo.blk_kind, ob_budget, w.theta, transfer=False,
                   device=dev.index, stream=stream, keep_dist=False, explicit_dist=True)
    ptr_t = torch.from_numpy(ob.ref_ptr).to(dev)
    ag_t = torch.from_numpy(ob.ref_agent).to(dev)
    by_t = torch.from_numpy(ob.obj_bytes).to(dev)
    ev = []
    dist_t = []

    def one(s, timed):
        agents.set_inputs_ptr(recs[s].data_ptr())
        agents.step(int(w.now[s]))
        if not dist_t:
            dist_t.append(agents.dist_tensor())  # the view exists after the first plan
        if timed:
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                 torch.cuda.Event(enable_timing=True))
            e[0].record(stream)
        object_min(dist_t[0], ptr_t, ag_t, by_t, objs.rec, obj_flags=flags[s], stream=stream)
        if timed:
            e[1].record(stream)
        objs.step(int(w.now[s]))
        if timed:
            e[2].record(stream)
            ev.append(e)

    for s in range(warm):
        one(s, False)
    torch.cuda.synchronize(dev)
    lc0 = agents.launch_count() + objs.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e8))
    t0.record(stream)
    for s in range(warm, T):
        one(s, True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1)
    om = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    op = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    hdr = objs.sync()
    launches = agents.launch_count() + objs.launch_count() - lc0 + steps  # + one object_min launch per step
    refs = int(ob.ref_ptr[-1])
    # object_min algorithmic bytes: CSR offsets 8 B + size 4 B + flags 4 B + record 16 B per object,
    # 4 B agent index + 4 B agent distance per reference
    om_bytes = 32 * ob.n + 8 * refs
    agents.close()
    objs.close()
    return {"value": ob.n * steps / (ms / 1e3), "unit": "object-plans/s",
            "workload": f"NEXT#1 shared objects: {n} C4 agents, {ob.n} objects (1 prompt prefix shared by all, "
                        f"{ob.n - 1 - n} persona adapters, {n} private KV-page objects), {refs} references",
            "ms_per_step": ms / steps, "includes": "agent plan + scalesim_object_min + object plan per step",
            "object_min_ms": om, "object_plan_ms": op,
            "object_min_GBs": om_bytes / (om / 1e3) / 1e9, "object_min_bytes": om_bytes,
            "last_object_plan": {"n_prefetch": hdr["n_prefetch"], "n_evict": hdr["n_evict"],
                                 "status": hdr["status"]},
            "gpu_launches": launches, "steps": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000, help="agents per GPU")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--eager", action="store_true", help="no CUDA graph")
    ap.add_argument("--no-transfer-leg", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=64)
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 replicas x budgets leg")
    ap.add_argument("--c5-replicas", type=int, default=64)
    ap.add_argument("--no-objects", action="store_true", help="skip the shared-object leg (NEXT #1)")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 planning + transfer overlap leg")
    ap.add_argument("--no-closed-loop", action="store_true", help="skip the closed-loop policy comparison (NEXT #3)")
    ap.add_argument("--no-sched", action="store_true", help="skip the load scheduler leg (NEXT #2)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the 1M..64M agent N-sweep")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_2601_21473_b200 import _lib
    from paper_2601_21473_b200.planner import Planner

    n = args.n
    W, K = args.warmup, args.steps
    T = WARM_IN + W + 2 * K  # K timed steps (eager, then per-kernel events), K graph-replayed steps: distinct buffers
    w = c4_shard(n, T, args.seed, rank)
    budget = w.budget
    nccl_id = None
    if world > 1:
        tot = torch.tensor([int(w.footprint.sum())], dtype=torch.int64, device=dev)
        dist.all_reduce(tot)
        budget = int(tot.item()) // 4
        obj = [None]
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            _lib.check(_lib.lib().scalesim_nccl_unique_id(buf), "scalesim_nccl_unique_id")
            obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    b = w.blocks
    # the headline context owns the GPU (SCALESIM_F_EXCLUSIVE: no cooperative-launch attribute,
    # include/scalesim.h); the default (cooperative) launch is timed beside it
    pl = Planner(n * world, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta,
                 transfer=False, device=local, shard=(rank * n, (rank + 1) * n), rank=rank, world=world,
                 nccl_id=nccl_id, keep_dist=False, exclusive=True)
    # all step records resident in HBM (T distinct 16 MB buffers, > L2)
    recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(T, -1)).to(dev)
    ptr = [recs[s].data_ptr() for s in range(T)]

    def eager_step(s):
        pl.set_inputs_ptr(ptr[s])
        pl.step(int(w.now[s]))

    for s in range(WARM_IN + W):
        eager_step(s)
    seq0 = pl.sync()["seq"]
    t_base = WARM_IN + W

    def steps(first, evs=None):
        for k in range(K):
            s = first + k
            pl.set_inputs_ptr(ptr[s])
            if evs:
                evs[0][k].record(pl.stream)
            pl.score(int(w.now[s]))
            pl.plan()
            if evs:
                evs[1][k].record(pl.stream)
            pl.transfer()
        pl.join()

    # (1) timed region: K steps launched eagerly through the step API (score + plan per step),
    # all enqueued while the GPU spins, so the device runs them back to back (programmatic
    # dependent launch overlaps each plan kernel's prologue with the previous one's tail)
    mode = "eager launches, K steps enqueued behind a spin kernel (device-timed; the host enqueues ahead)"
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        with torch.cuda.stream(pl.stream):
            torch.cuda._sleep(int(2e9 * 0.05 + K * 2e5))
        lc0 = pl.launch_count()
        t0.record(pl.stream)
        steps(t_base)
        t1.record(pl.stream)
        launches = pl.launch_count() - lc0
        sampler.poll_until(t1)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    hdr = pl.sync()
    # integrity: the device completed exactly K plans in the timed region
    assert hdr["seq"] - seq0 == K, f"timed region ran {hdr['seq'] - seq0} plans, expected {K}"
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / K
    value = n * world * K / (ms / 1e3)

    # (1a) the default launch mode (cooperative attribute, any context may run concurrently
    # with other kernels): the same K steps on a second, non-exclusive context
    coop_ms = None
    if world == 1:
        pc = Planner(n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta, transfer=False,
                     device=local, keep_dist=False)
        for s in range(WARM_IN + W):
            pc.set_inputs_ptr(ptr[s])
            pc.step(int(w.now[s]))
        torch.cuda.synchronize(dev)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(pc.stream):
            torch.cuda._sleep(int(2e9 * 0.05 + K * 2e5))
        c0.record(pc.stream)
        for k in range(K):
            pc.set_inputs_ptr(ptr[t_base + k])
            pc.step(int(w.now[t_base + k]))
        c1.record(pc.stream)
        torch.cuda.synchronize(dev)
        coop_ms = c0.elapsed_time(c1) / K
        pc.close()

    # (1b) the same K-step loop captured once as a CUDA graph and replayed (next K buffers):
    # reported beside the eager number, not as the value
    graph_ms = None
    if not args.eager:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=pl.stream):
                steps(t_base + K)
            torch.cuda.synchronize(dev)
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            with torch.cuda.stream(pl.stream):
                g0.record(pl.stream)
                graph.replay()
                g1.record(pl.stream)
            torch.cuda.synchronize(dev)
            graph_ms = g0.elapsed_time(g1) / K
            if world > 1:
                t = torch.tensor([graph_ms], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                graph_ms = float(t.item())
            del graph
        except Exception as e:
            sys.stderr.write(f"graph capture failed ({e})\n")
            torch.cuda.synchronize(dev)
    hdr = pl.sync()

    # (2) the dominant kernel's launch duration with CUDA events on the launching stream:
    # K steps (the timed region's buffers again), enqueued while the GPU spins, events around each
    # step's plan launches
    fused = pl.fused
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(pl.stream):
        torch.cuda._sleep(int(2e9 * 0.05 + K * 2e5))
    steps(t_base, (ev_a, ev_b))
    torch.cuda.synchronize(dev)
    ms_kern = [ev_a[k].elapsed_time(ev_b[k]) for k in range(K)]
    hdr2 = pl.sync()
    assert hdr2["seq"] - hdr["seq"] == K

    # ---- e2e: the same metric through the host entry point (host buffers, copies inside)
    e2e_k = min(args.e2e_steps, K)
    rec_pinned = torch.from_numpy(np.ascontiguousarray(w.rec[t_base:t_base + e2e_k])).pin_memory()
    rec_host = [rec_pinned[k].numpy() for k in range(e2e_k)]
    pf = np.zeros(n, np.uint32)
    ev = np.zeros(n, np.uint32)
    if world > 1:
        dist.barrier()
    # the changed records of each step (the simulation emits them as its agents act; computed
    # before the region), pinned
    upd = [None]
    for k in range(1, e2e_k):
        ch = np.nonzero(np.any(w.rec[t_base + k] != w.rec[t_base + k - 1], axis=1))[0].astype(np.uint32)
        upd.append((torch.from_numpy(ch + np.uint32(rank * n)).pin_memory().numpy(),  # global ids
                    torch.from_numpy(np.ascontiguousarray(w.rec[t_base + k][ch])).pin_memory().numpy()))

    def e2e_loop(mode):
        """e2e_k steps through the host entry points; returns (seconds, h2d bytes, d2h bytes).
        sync: scalesim_step_host alone (copy, plan, read back, one step at a time).
        full: scalesim_stage_host starts step k+1's record copy (copy engine, its own stream)
        before step k's scalesim_step_host, whose plan waits for its staged copy on the device.
        updates: after step 0's whole records, each step sends only its changed records
        (scalesim_stage_updates one step ahead + scalesim_step_updates).  Every step's H2D and
        its header + lists D2H are inside the region."""
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        hb = db = 0
        if mode == "full":
            pl.stage_host(rec_host[0])
        if mode == "submit":  # three steps in flight: steps k+1, k+2 copy and plan while k is collected
            h = pl.step_host(int(w.now[t_base]), rec_host[0], None, pf, ev)
            hb += rec_host[0].nbytes
            db += 128 + 4 * (h["n_prefetch"] + h["n_evict"])
            for k in range(1, min(3, e2e_k)):
                pl.submit_updates(int(w.now[t_base + k]), *upd[k])
            for k in range(1, e2e_k):
                if k + 2 < e2e_k:
                    pl.submit_updates(int(w.now[t_base + k + 2]), *upd[k + 2])
                h = pl.collect(pf, ev)
                hb += upd[k][0].nbytes + upd[k][1].nbytes
                db += 128 + 4 * (h["n_prefetch"] + h["n_evict"])
        for k in range(e2e_k if mode != "submit" else 0):
            if mode == "updates" and k > 0:
                if k + 1 < e2e_k:
                    pl.stage_updates(*upd[k + 1])
                h = pl.step_updates(int(w.now[t_base + k]), upd[k][0], upd[k][1], pf, ev)
                hb += upd[k][0].nbytes + upd[k][1].nbytes
            else:
                if mode == "full" and k + 1 < e2e_k:
                    pl.stage_host(rec_host[k + 1])
                h = pl.step_host(int(w.now[t_base + k]), rec_host[k], None, pf, ev)
                hb += rec_host[k].nbytes
                if mode == "updates" and e2e_k > 1:
                    pl.stage_updates(*upd[1])
            db += 128 + 4 * (h["n_prefetch"] + h["n_evict"])
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el, hb, db

    # each mode once untimed first (the staging buffers, streams and the host-mapped error word
    # are allocated on first use), then timed
    el_s, _, _ = [e2e_loop("sync") for _ in range(2)][-1]
    el_f, h2d_f, _ = [e2e_loop("full") for _ in range(2)][-1]
    el_u, _, _ = [e2e_loop("updates") for _ in range(2)][-1]
    el_e, h2d_b, d2h_b = [e2e_loop("submit") for _ in range(2)][-1]
    e2e = {"value": n * world * e2e_k / el_e, "unit": "agent-plans/s", "h2d_bytes_per_step": h2d_b // e2e_k,
           "d2h_bytes_per_step": d2h_b // e2e_k, "steps": e2e_k,
           "api": "step 0 whole records (scalesim_step_host), then each step's changed records (ids + "
                  "16-byte records, pinned) by scalesim_submit_updates, three steps in flight, header + "
                  "lists of every step back through scalesim_collect; host-timed, all copies inside",
           "sync_updates_value": n * world * e2e_k / el_u,
           "sync_updates_api": "scalesim_stage_updates one step ahead + scalesim_step_updates (synchronous)",
           "changed_per_step": float(np.mean([len(u[0]) for u in upd[1:]])) if e2e_k > 1 else None,
           "whole_records_value": n * world * e2e_k / el_f, "whole_records_h2d_bytes_per_step": h2d_f // e2e_k,
           "whole_records_h2d_GBs": h2d_f / el_f / 1e9,
           "whole_records_api": "scalesim_stage_host(records of step t+1) + scalesim_step_host(step t)",
           "synchronous_value": n * world * e2e_k / el_s,
           "synchronous_api": "scalesim_step_host alone (16 MB records in, plan, header + lists out, one step at a time)"}

    pl.close()
    c5 = None
    if not args.no_c5:
        if world > 1:
            dist.barrier()
        r5 = c5_leg(torch, dev, rank, world, replicas=args.c5_replicas)
        if world > 1:
            t = torch.tensor([r5["ms"], r5["agents_per_step"]], dtype=torch.float64, device=dev)
            mx = t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = t.clone()
            dist.all_reduce(sm)
            r5["ms"], r5["agents_per_step"] = float(mx[0].item()), int(sm[1].item())
        c5_gbs = r5["agents_per_step"] * BYTES_PER_AGENT_STEP / (r5["ms"] / r5["steps"] / 1e3) / 1e9
        c5 = {"value": r5["agents_per_step"] * r5["steps"] / (r5["ms"] / 1e3), "unit": "agent-plans/s",
              "roofline": {"bound": "hbm", "achieved": c5_gbs, "peak": peaks()["hbm_gbs"], "unit": "GB/s",
                           "frac": c5_gbs / peaks()["hbm_gbs"], "frac_8TBs": c5_gbs / 8000.0,
                           "algorithmic_bytes_per_step": r5["agents_per_step"] * BYTES_PER_AGENT_STEP,
                           "timing": "the step's launches (ceil(instances / 148) batched plan kernels) on one stream, "
                                     "CUDA events around the timed steps"},
              "workload": f"c5: {args.c5_replicas} replicas x 9 budgets (10..90%) of the C2 shape (10k agents), "
                          f"instances sharded over {world} GPU(s), scalesim_step_batch",
              "instances_per_gpu": r5["instances"], "steps": r5["steps"], "ms_per_step": r5["ms"] / r5["steps"],
              "gpu_launches": r5["launches"]}
    sweep = None
    if not args.no_sweep and rank == 0:
        sweep = sweep_leg(torch, dev, peaks()["hbm_gbs"])
    objects = None
    if not args.no_objects and rank == 0:
        objects = objects_leg(torch, dev)
    c3 = None
    if not args.no_c3 and rank == 0:
        c3 = c3_leg(torch, dev)
    cl = None
    if not args.no_closed_loop and rank == 0:
        cl = closed_loop_leg(dev)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk = peaks()
    iso_ms = float(np.mean(ms_kern))  # events bracketing each launch (breaks the launch overlap)
    one_launch = fused and launches == K
    # the fused path launches exactly one kernel per step (gpu_launches == K): its average launch
    # duration in the timed region is the region's event time / K, measured on the stream it runs on
    kern_ms = ms_per_step if one_launch else iso_ms
    if fused:
        # one persistent kernel scores and plans the step: its launch is the dominant kernel
        per_agent = BYTES_PER_AGENT_STEP
        kname = "k_fused_plan (score+select+cut+emit+list sort: one launch per step)"
    else:
        per_agent = BYTES_PER_AGENT_STEP
        kname = "multi-kernel plan (all launches of scalesim_score + scalesim_plan)"
    achieved = n * per_agent / (kern_ms / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_traffic.json")))
        if prof.get("kernel_prefix") and kname.startswith(prof["kernel_prefix"]):
            traffic = prof["dram_bytes_per_launch"]
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "algorithmic_bytes_per_launch": n * per_agent,
            "kernel_ms": kern_ms,
            "kernel_share_of_step": kern_ms / ms_per_step,
            "timing": ("timed region's CUDA events on the planner stream / K (one launch of this kernel per "
                       "step, gpu_launches == steps)") if one_launch else
                      "CUDA events around each step's launches on the planner stream, K steps pre-enqueued",
            "isolated_launch_ms": iso_ms, "isolated_launch_ms_p10_p90": [float(np.percentile(ms_kern, 10)),
                                                                         float(np.percentile(ms_kern, 90))],
            "isolated_launch_note": "events bracketing each launch separately (no overlap with the previous "
                                    "launch's tail)",
            "step_frac": n * BYTES_PER_AGENT_STEP / (ms_per_step / 1e3) / 1e9 / pk["hbm_gbs"],
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)" if not pk.get("_fallback")
            else "fallback 6650"}
    line = {"metric": "agent-plans/sec (1M agents, 1/2/4/8 B200) % HBM roofline; transfer GB/s vs host link",
            "value": value, "unit": "agent-plans/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c4: 1M independent AgentSociety-shaped agents per GPU (C3 footprints, logical "
                                   "sizes), budget 25% of agent memory, theta 4, ~5% active/step",
                       "n_agents_per_gpu": n, "n_agents": n * world, "parallelism": f"id-shard x{world}",
                       "l2": f"{K} distinct 16 MB record buffers (> 126 MB L2)", "timing": mode,
                       "graph_replay_ms_per_step": graph_ms,
                       "launch_mode": "SCALESIM_F_EXCLUSIVE (device dedicated to the planner: no cooperative "
                                      "attribute, programmatic dependent launch)",
                       "cooperative_mode_ms_per_step": coop_ms,
                       "last_plan": {k: hdr[k] for k in ("n_prefetch", "n_evict", "cut_bits", "status")}},
            "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": sampler.result()}
    if c5 is not None:
        line["c5"] = c5
    if sweep is not None:
        line["n_sweep"] = sweep
    if objects is not None:
        line["objects"] = objects
    if c3 is not None:
        line["c3"] = c3
    if cl is not None:
        line["closed_loop"] = cl
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    if not args.no_transfer_leg:
        lp = link_peak(torch, dev)
        tl = transfer_leg(torch, dev, args.seed)
        tl["link"] = lp
        # link-bound lower bound of a step's transfer: loads and write-backs overlapped
        # (full-duplex PCIe), each at the cudaMemcpy peak measured in this run
        ideal_s = max(tl["h2d_bytes_per_step"] / (lp["h2d_GBs"] * 1e9), tl["d2h_bytes_per_step"] / (lp["d2h_GBs"] * 1e9))
        tl["frac_of_link"] = ideal_s / max(tl["bytes_per_step"] / (tl["GBs"] * 1e9), 1e-12)
        tl["frac_definition"] = "max(h2d/h2d_peak, d2h/d2h_peak) / measured transfer time per step"
        line["transfer"] = tl
        if not args.no_sched:
            line["scheduler"] = sched_leg(torch, dev, lp)
    line["cpu"] = {"cores": os.cpu_count()}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
