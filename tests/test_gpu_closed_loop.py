"""GPU closed loop (NEXT #3): the invocation-distance policy and the reactive LRU baseline
(scalesim_lru_records + explicit-distance planning, reading R20) step through a trace in the
library; per-step misses and bytes equal the oracle's closed loop."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import rec_of

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
