"""Pins of the shared-object oracle (reading R19) and of explicit
distances: the paper's example, S:269-270's properties, the two properties that make a
minimum unique (lower bound + attained), and the special case where every object is one
agent's private memory (object planning = agent planning)."""
import json
import os

import numpy as np
import pytest

import oracle
import tracegen as tg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.uint64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    return ptr, np.array([a for x in lists for a in x], np.uint32)


def test_paper_shared_object_example():
    g = json.load(open(os.path.join(GOLD, "shared_object_example.json")))
    ptr, ag = _csr(g["objects"])
    d, st = oracle.object_min(np.array(g["agent_dist"], np.float32), ptr, ag)
    exp = np.array([np.inf if x == "inf" else x for x in g["expected"]], np.float32)
    assert st == 0 and np.array_equal(d, exp)


def test_min_properties_random():
    """d(o) <= d(a) for every referrer a (lower bound) and d(o) = d(a) for some referrer
    (attained); +inf exactly when the object has no referrer."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(1, 60))
        dist = rng.choice([0.0, 1.0, 2.0, 3.5, 7.0, np.inf], n).astype(np.float32)
        m = rng.random(n) < 0.3
        dist[m] = (rng.random(int(m.sum())) * 50).astype(np.float32)
        lists = [list(rng.integers(0, n, int(rng.integers(0, 6)))) for _ in range(int(rng.integers(1, 40)))]
        ptr, ag = _csr(lists)
        d, st = oracle.object_min(dist, ptr, ag)
        assert st == 0
        for o, refs in enumerate(lists):
            if not refs:
                assert d[o] == np.inf
            else:
                assert all(d[o] <= dist[a] for a in refs)
                assert any(d[o] == dist[a] for a in refs)


def test_min_monotone_when_an_agent_gets_closer():
    """agent distance drops 5 -> 0: all its objects' distances <= previous values."""
    rng = np.random.default_rng(6)
    n = 50
    dist = rng.integers(1, 20, n).astype(np.float32)
    lists = [list(rng.integers(0, n, int(rng.integers(1, 5)))) for _ in range(80)]
    ptr, ag = _csr(lists)
    before, _ = oracle.object_min(dist, ptr, ag)
    dist2 = dist.copy()
    dist2[7] = 0.0
    after, _ = oracle.object_min(dist2, ptr, ag)
    assert np.all(after <= before)
    for o, refs in enumerate(lists):
        if 7 in refs:
            assert after[o] == 0.0


def test_bad_references_and_values():
    ptr, ag = _csr([[0, 5], [1], [2]])
    d, st = oracle.object_min(np.array([3.0, np.nan, -0.0], np.float32), ptr, ag)
    assert st & oracle.ST_BAD_RECORD
    assert d[0] == 3.0 and d[1] == np.inf and d[2] == 0.0 and not np.signbit(d[2])


def test_explicit_distance_reading():
    vals = np.array([0.0, 1.5, 7.0, np.inf], np.float32)
    rec = np.zeros((6, 4), np.uint32)
    rec[:4, 0] = vals.view(np.uint32)
    rec[4, 0] = 0x80000000  # -0
    rec[5, 0] = np.float32(-2.0).view(np.uint32)
    d, st = oracle.explicit_dist(rec)
    assert np.array_equal(d[:4], vals) and d[4] == 0.0 and not np.signbit(d[4])
    assert d[5] == np.inf and st == oracle.ST_BAD_RECORD


@pytest.mark.parametrize("seed", [1, 2])
def test_private_objects_plan_like_agents(seed):
    """Special case: each object is one agent's private memory (one referrer, same bytes):
    object distances = agent distances and the object plan = the agent plan."""
    w = tg.config_c2(seed=seed, steps=6, n=800, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    n = w.n
    ptr = np.arange(n + 1, dtype=np.uint64)
    ag = np.arange(n, dtype=np.uint32)
    res_a = np.zeros(n, np.uint8)
    res_o = np.zeros(n, np.uint8)
    for s in range(w.steps):
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        pa = oracle.plan(w.rec[s], d, res_a, w.theta, w.budget)
        do, st = oracle.object_min(d, ptr, ag)
        assert st == 0 and np.array_equal(do.view(np.uint32), d.view(np.uint32))
        orec = np.zeros((n, 4), np.uint32)
        orec[:, 0] = do.view(np.uint32)
        orec[:, 1] = w.rec[s][:, 1]
        dx, _ = oracle.explicit_dist(orec)
        po = oracle.plan(orec, dx, res_o, w.theta, w.budget)
        for k in ("prefetch", "evict", "resident"):
            assert np.array_equal(pa[k], po[k]), (s, k)
        assert pa["cut_bits"] == po["cut_bits"] and pa["bytes_h2d"] == po["bytes_h2d"]
        res_a, res_o = pa["resident"], po["resident"]


def test_gen_objects_structure():
    o = tg.gen_objects(1000, seed=3)
    assert o.ref_ptr[-1] == len(o.ref_agent) == 3000
    assert np.diff(o.ref_ptr.astype(np.int64))[0] == 1000  # the prompt is shared by every agent
    assert np.all(np.diff(o.ref_ptr.astype(np.int64))[-1000:] == 1)  # private pages
    assert np.all(o.obj_bytes % tg.PAGE_BYTES == 0)
