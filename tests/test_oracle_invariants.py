"""Invariant pins of the oracle on generated traces (north star
invariants) and of its paged-arena bookkeeping.  No GPU."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import keys_of, rec_of


def check_plan_invariants(rec, d, res_in, theta, budget, p):
    n = rec.shape[0]
    fp = rec[:, 1].astype(np.int64)
    cls = (rec[:, 2] >> 2) & 3
    th = np.where(cls < 3, theta[np.minimum(cls, 2)], 0)
    elig = (res_in != 0) | (d == 0) | (d < th)
    kept = p["resident"].astype(bool)
    keys = keys_of(d, np.arange(n))
    # capacity safety: resident bytes <= budget
    assert fp[kept].sum() <= budget
    assert p["kept_bytes"] == fp[kept].sum()
    # only eligible agents are kept; residents are always eligible (R4)
    assert not np.any(kept & ~elig)
    # "the evicted set never outranks the kept set": kept is a prefix of the eligible order
    if kept.any() and (elig & ~kept).any():
        assert keys[kept].max() < keys[elig & ~kept].min()
    # maximality: the first eligible agent left out does not fit (R3)
    if (elig & ~kept).any():
        first = np.argmin(np.where(elig & ~kept, keys, np.iinfo(np.uint64).max))
        assert fp[kept].sum() + fp[first] > budget
        assert p["cut_bits"] == int(np.float32(d[first]).view(np.uint32))
    else:
        assert p["cut_bits"] == 0xFFFFFFFF
    # conservation: resident' = (resident \ evict) U prefetch
    new = res_in.astype(bool).copy()
    new[p["evict"]] = False
    new[p["prefetch"]] = True
    assert np.array_equal(new, kept)
    # prefetch = the top |prefetch| non-resident eligible agents, ascending key (R14)
    cand = np.nonzero(elig & (res_in == 0))[0]
    cand = cand[np.argsort(keys[cand], kind="stable")]
    assert np.array_equal(p["prefetch"], cand[:len(p["prefetch"])])
    ek = keys[p["evict"]]
    assert np.all(ek[:-1] > ek[1:])  # evict: descending key
    assert p["bytes_h2d"] == fp[p["prefetch"]].sum()
    # pinning: an active (d == 0) agent is only left out when memory is insufficient
    zero_out = np.any((d == 0) & ~kept)
    assert bool(p["status"] & oracle.ST_INSUFFICIENT) == bool(zero_out)
    # prefetch safety: no evicted agent has a smaller key than a prefetched one
    if len(p["prefetch"]) and len(p["evict"]):
        assert keys[p["prefetch"]].max() < keys[p["evict"]].min()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c2_trace_invariants_and_idempotence(seed):
    w = tg.config_c2(seed=seed, steps=48, n=3000)
    res = np.zeros(w.n, np.uint8)
    for s in range(w.steps):
        d, st = oracle.score(w.rec[s], None, w.now[s])
        assert st == 0
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        check_plan_invariants(w.rec[s], d, res, w.theta, w.budget, p)
        # idempotence: re-planning from the kept set with the same distances changes nothing
        p2 = oracle.plan(w.rec[s], d, p["resident"], w.theta, w.budget)
        assert len(p2["prefetch"]) == 0 and len(p2["evict"]) == 0
        res = p["resident"]


def test_c3_mixed_classes_invariants():
    w = tg.config_c3(seed=1, steps=3, n=3000, budget=int(3000 * 3.4e6 * 0.235))
    res = np.zeros(w.n, np.uint8)
    for s in range(w.steps):
        d, st = oracle.score(w.rec[s], w.kin[s], w.now[s], w.hop_scale)
        assert st == 0
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        check_plan_invariants(w.rec[s], d, res, w.theta, w.budget, p)
        res = p["resident"]


def test_budget_nesting():
    """R*(B) is a subset of R*(B') for B <= B' (the C5 sweep axis)."""
    w = tg.config_c2(seed=7, steps=1, n=2000)
    d, _ = oracle.score(w.rec[0], None, w.now[0])
    rng = np.random.default_rng(0)
    res = (rng.random(w.n) < 0.2).astype(np.uint8)
    total = int(w.rec[0, :, 1].astype(np.int64).sum())
    prev = None
    for pct in range(10, 100, 10):
        p = oracle.plan(w.rec[0], d, res, np.full(3, np.inf, np.float32), total * pct // 100)
        kept = p["resident"].astype(bool)
        if prev is not None:
            assert not np.any(prev & ~kept)
        prev = kept


def test_empty_and_degenerate():
    # no agents
    p = oracle.plan(np.zeros((0, 4), np.uint32), np.zeros(0, np.float32), np.zeros(0, np.uint8),
                    np.zeros(3, np.float32), 10)
    assert p["prefetch"].size == 0 and p["cut_bits"] == 0xFFFFFFFF
    # zero budget: nothing kept; actives flagged
    rec = rec_of([dict(phase=tg.PH_GENERATING), dict(d=2)])
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.array([0, 1], np.uint8), np.full(3, 9.0, np.float32), 0)
    assert p["resident"].sum() == 0 and p["evict"].tolist() == [1]
    assert p["status"] & oracle.ST_INSUFFICIENT
    # zero-size agents: kept only inside the prefix (R3 strict prefix)
    rec = rec_of([dict(d=1, fp=5), dict(d=2, fp=0), dict(d=3, fp=9), dict(d=4, fp=0)])
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.zeros(4, np.uint8), np.full(3, 9.0, np.float32), 6)
    assert p["resident"].tolist() == [1, 1, 0, 0]
    # everything fits: cut_bits sentinel and rem = B - kept
    p = oracle.plan(rec, d, np.zeros(4, np.uint8), np.full(3, 9.0, np.float32), 100)
    assert p["cut_bits"] == 0xFFFFFFFF and p["cut_rem"] == 100 - 14


# ----------------------------------------------------------------------------------------
# Paged arena

PG = tg.PAGE_BYTES


def test_pages_hand_example():
    """FIFO pool: evicted pages are appended in evict order, block order, page order, then the
    prefetched agents pop pages from the head in prefetch order."""
    blocks = tg.make_blocks([[tg.KIND_LORA, tg.KIND_KV], [tg.KIND_KV], [tg.KIND_LORA, tg.KIND_HIST]],
                            [[2 * PG, PG], [PG], [PG, PG]])
    m = oracle.OracleMem(blocks.blk_ptr, blocks.blk_size, blocks.blk_host_off, blocks.blk_kind, PG, 5,
                         resident_init=np.array([1, 0, 0], np.uint8))
    assert m.page_table().tolist() == [0, 1, 2] + [0xFFFFFFFF] * 3
    rec = rec_of([dict(d=9, fp=3 * PG, dirty=1), dict(phase=tg.PH_WAITING, fp=PG), dict(d=1, fp=2 * PG)])
    out = m.apply(rec, prefetch=[2, 1], evict=[0])
    off = blocks.blk_host_off
    # dirty agent 0: its KV block (page 2) is written back, its LoRA block is not (R13)
    assert out["d2h_host"].tolist() == [int(off[1])] and out["d2h_page"].tolist() == [2]
    assert out["bytes_d2h"] == PG
    # pool after release: head=3 -> pages 3, 4, then the released 0, 1, 2
    assert out["h2d_page"].tolist() == [3, 4, 0]
    assert out["h2d_host"].tolist() == [int(off[3]), int(off[4]), int(off[2])]
    assert out["bytes_h2d"] == 3 * PG
    assert m.page_table().tolist() == [0xFFFFFFFF] * 3 + [0, 3, 4]


def test_pages_conservation_on_trace():
    w = tg.config_c2(seed=5, steps=40, n=400, lora=4 * PG, kv=PG)
    nb_pages = w.budget // PG + 1
    res = np.zeros(w.n, np.uint8)
    b = w.blocks
    m = oracle.OracleMem(b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, PG, nb_pages)
    page_first = np.concatenate([[0], np.cumsum(b.blk_size // PG)]).astype(np.int64)
    agent_of_page = np.repeat(np.repeat(np.arange(w.n), np.diff(b.blk_ptr).astype(np.int64)),
                              (b.blk_size // PG).astype(np.int64))
    for s in range(w.steps):
        d, _ = oracle.score(w.rec[s], None, w.now[s])
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        out = m.apply(w.rec[s], p["prefetch"], p["evict"])
        assert out["status"] == 0
        assert out["bytes_h2d"] == p["bytes_h2d"]
        dirty = (w.rec[s, :, 2] >> 4) & 1
        wb = 0
        for a in p["evict"]:
            if dirty[a]:
                for blk in range(int(b.blk_ptr[a]), int(b.blk_ptr[a + 1])):
                    wb += int(b.blk_size[blk]) if b.blk_kind[blk] != tg.KIND_LORA else 0
        assert out["bytes_d2h"] == wb
        res = p["resident"]
        pt = m.page_table()
        valid = pt != 0xFFFFFFFF
        assert np.array_equal(valid, res[agent_of_page].astype(bool))
        head, tail, ring = m.pool()
        free = [ring[k % nb_pages] for k in range(head, tail)]
        allp = np.sort(np.concatenate([pt[valid], np.array(free, np.uint32)]))
        assert np.array_equal(allp, np.arange(nb_pages))
        assert len(out["h2d_page"]) == sum(int(w.rec[s, a, 1]) // PG for a in p["prefetch"])
    del page_first
