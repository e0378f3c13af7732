"""GPU closed loop (NEXT #3): the invocation-distance policy and the reactive LRU baseline
(scalesim_lru_records + explicit-distance planning, reading R20) step through a trace in the
library; per-step misses and bytes equal the oracle's closed loop."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import rec_of, two_agent_overlap_records

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


def _canonical_records(trace, n_agents):
    T = len(trace)
    recs = []
    for t in range(T):
        agents = []
        for a in range(n_agents):
            nxt = next((u for u in range(t, T) if trace[u] == a), None)
            if nxt is None:
                agents.append(dict(phase=tg.PH_IDLE))
            elif nxt == t:
                agents.append(dict(phase=tg.PH_WAITING))
            else:
                agents.append(dict(d=nxt - t))
        recs.append(rec_of(agents, now=t))
    return np.stack(recs)


def test_canonical_trace_on_gpu():
    """1,2,3,1,2,3 with capacity 2: LRU 6 misses, invocation distance 4."""
    from paper_2601_21473_b200 import closed_loop
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "canonical_trace.json")))
    recs = _canonical_records(g["trace"], 4)
    blocks = tg.make_blocks([[tg.KIND_KV]] * 4, [[tg.PAGE_BYTES]] * 4)
    budget = g["capacity"] * tg.PAGE_BYTES
    recs[:, :, 1] = tg.PAGE_BYTES
    args = (recs, np.arange(len(recs), dtype=np.int64), blocks.blk_ptr, blocks.blk_size, blocks.blk_host_off,
            blocks.blk_kind, budget, np.zeros(3, np.float32))
    lru = closed_loop.run(*args, policy="lru")
    dist = closed_loop.run(*args, policy="distance")
    assert lru["misses"].sum() == g["expected_lru_misses"]
    assert dist["misses"].sum() == g["expected_distance_misses"]


def _oracle_loop(w, policy):
    res = np.zeros(w.n, np.uint8)
    last = np.full(w.n, 0xFFFFFFFF, np.uint32)
    out = []
    for s in range(w.steps):
        if policy == "lru":
            rec = oracle.lru_records(w.rec[s], int(w.now[s]), last)
            d, _ = oracle.explicit_dist(rec)
            th = np.zeros(3, np.float32)
        else:
            rec = w.rec[s]
            d, _ = oracle.score(rec, None, int(w.now[s]))
            th = w.theta
        p = oracle.plan(rec, d, res, th, w.budget)
        pf = p["prefetch"]
        demand = pf[d[pf] == 0.0]
        out.append((len(demand), int(w.rec[s][demand, 1].astype(np.int64).sum()), p["bytes_h2d"], len(pf),
                    len(p["evict"])))
        res = p["resident"]
    return np.array(out)


@pytest.mark.parametrize("policy", ["distance", "lru"])
def test_closed_loop_vs_oracle(policy):
    from paper_2601_21473_b200 import closed_loop
    w = tg.config_c2(seed=5, steps=30, n=2000, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    b = w.blocks
    got = closed_loop.run(w.rec, w.now, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                          policy=policy)
    exp = _oracle_loop(w, policy)
    assert np.array_equal(got["misses"], exp[:, 0])
    assert np.array_equal(got["miss_bytes"], exp[:, 1])
    assert np.array_equal(got["loaded_bytes"], exp[:, 2])
    assert np.array_equal(got["n_prefetch"], exp[:, 3]) and np.array_equal(got["n_evict"], exp[:, 4])


def test_prefetch_overlap_closed_form():
    """with B's action longer than transfer_time(A), the scalesim preset's stall for A's
    next request is 0 and the reactive presets' is transfer_time(A) exactly."""
    from paper_2601_21473_b200 import closed_loop
    F = 1000 * tg.PAGE_BYTES
    recs = two_agent_overlap_records(F)
    blocks = tg.make_blocks([[tg.KIND_KV]] * 2, [[F]] * 2)
    link, step_s = 55.0, 0.05
    T_A = F / (link * 1e9)
    assert T_A < 5 * step_s
    args = (recs, np.arange(len(recs), dtype=np.int64), blocks.blk_ptr, blocks.blk_size, blocks.blk_host_off,
            blocks.blk_kind, F, np.full(3, 10.0, np.float32))
    out = {p: closed_loop.run(*args, policy=p, link_GBs=link, step_s=step_s)
           for p in ("scalesim", "hicache_like", "sglang_like")}
    assert out["scalesim"]["stall_s"][7] == 0.0
    assert abs(out["hicache_like"]["stall_s"][7] - T_A) <= 1e-12 * T_A, out["hicache_like"]["stall_s"]
    for p in ("hicache_like", "sglang_like"):
        assert out[p]["misses"][7] == 1
    # sglang_like: A's KV was dropped when B took the slot: recomputed, not moved
    assert out["sglang_like"]["recompute_bytes"][7] == F and out["sglang_like"]["stall_s"][7] == 0.0
    assert out["scalesim"]["misses"][7] == 0 and out["scalesim"]["n_prefetch"][2] == 1
    # the cold starts (steps 0 and 1) stall every preset by one transfer
    for p in out:
        assert abs(out[p]["stall_s"][0] - T_A) <= 1e-12 * T_A and abs(out[p]["stall_s"][1] - T_A) <= 1e-12 * T_A


def test_sglang_like_drops_and_recomputes_kv():
    """sglang_like: evicted KV / history is not written back, its reload is recompute;
    hicache_like writes dirty KV back and reloads it over the link."""
    from paper_2601_21473_b200 import closed_loop
    w = tg.config_c2(seed=5, steps=30, n=2000, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    b = w.blocks
    args = (w.rec, w.now, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta)
    hi = closed_loop.run(*args, policy="hicache_like")
    sg = closed_loop.run(*args, policy="sglang_like")
    assert np.array_equal(hi["misses"], sg["misses"])  # the same LRU plans
    assert sg["writeback_bytes"].sum() == 0 and hi["writeback_bytes"].sum() > 0
    assert sg["recompute_bytes"].sum() > 0
    assert np.array_equal(sg["loaded_bytes"] + sg["recompute_bytes"], hi["loaded_bytes"])
