"""world > 1 on one GPU: the ranks of a world (SCALESIM_F_LOOPBACK
contexts, one contiguous id shard each) stepped by scalesim_step_group give plan(world) ==
plan(1) == oracle, bit for bit: every rank's lists are the global lists restricted to its
shard (same order), its residency the global residency of its shard, and the world-wide header
fields (D*, rem, kept bytes, eligible agents, INSUFFICIENT) the global ones.  Covers the
fast list placement, a tie group cut inside a later rank's shard, the multi-level select /
two-barrier list path, and physical page transfers per rank."""
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


def shard_blocks(b, lo, hi):
    p0, p1 = int(b.blk_ptr[lo]), int(b.blk_ptr[hi])
    return (b.blk_ptr[lo:hi + 1] - b.blk_ptr[lo], b.blk_size[p0:p1], b.blk_host_off[p0:p1], b.blk_kind[p0:p1])


def run_world(w, cuts, steps=None, transfer=False, resident_init=None, expect_paths=None):
    import torch
    from gpu_harness import fill_pattern
    from paper_2601_21473_b200.planner import Planner, step_group
    G = len(cuts) - 1
    stream = torch.cuda.Stream()
    ranks = []
    host = None
    if transfer:
        host = torch.empty(int(w.blocks.host_bytes), dtype=torch.uint8, pin_memory=True)
        fill_pattern(host)
    for r in range(G):
        lo, hi = cuts[r], cuts[r + 1]
        bp, bs, bo, bk = shard_blocks(w.blocks, lo, hi)
        ri = None if resident_init is None else resident_init[lo:hi]
        pages = (w.budget + w.page_bytes - 1) // w.page_bytes
        ranks.append(Planner(w.n, bp, bs, bo, bk, w.budget, w.theta, hop_scale=w.hop_scale, transfer=transfer,
                             page_bytes=w.page_bytes, host_arena=host, dev_bytes=max(pages, 1) * w.page_bytes,
                             shard=(lo, hi), rank=r, world=G, loopback=True, stream=stream, keep_dist=False,
                             resident_init=ri))
        assert ranks[-1].fused
    res = np.zeros(w.n, np.uint8) if resident_init is None else np.asarray(resident_init, np.uint8).copy()
    oms = None
    if transfer:
        oms = []
        for r in range(G):
            lo, hi = cuts[r], cuts[r + 1]
            bp, bs, bo, bk = shard_blocks(w.blocks, lo, hi)
            pages = max((w.budget + w.page_bytes - 1) // w.page_bytes, 1)
            oms.append(oracle.OracleMem(bp, bs, bo, bk, w.page_bytes, pages, resident_init=res[lo:hi]))
    steps = range(w.steps) if steps is None else steps
    for s in steps:
        rec = w.rec[s]
        for r, pl in enumerate(ranks):
            pl.set_records(rec[cuts[r]:cuts[r + 1]])
        step_group(ranks, int(w.now[s]))
        d, st = oracle.score(rec, None, int(w.now[s]), w.hop_scale)
        p = oracle.plan(rec, d, res, w.theta, w.budget)
        for r, pl in enumerate(ranks):
            lo, hi = cuts[r], cuts[r + 1]
            hdr = pl.sync()
            pf, ev = pl.lists(hdr)
            mpf = (p["prefetch"] >= lo) & (p["prefetch"] < hi)
            mev = (p["evict"] >= lo) & (p["evict"] < hi)
            assert np.array_equal(pf, p["prefetch"][mpf]), (s, r, pf[:8], p["prefetch"][mpf][:8])
            assert np.array_equal(ev, p["evict"][mev]), (s, r, ev[:8], p["evict"][mev][:8])
            assert np.array_equal(pl.resident(), p["resident"][lo:hi]), (s, r)
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"], (s, r, hdr, p["cut_bits"])
            assert hdr["kept_bytes"] == p["kept_bytes"] and hdr["n_eligible"] == p["n_eligible"], (s, r)
            assert (hdr["status"] & oracle.ST_INSUFFICIENT) == (p["status"] & oracle.ST_INSUFFICIENT), (s, r)
            fp = rec[:, 1].astype(np.int64)
            assert hdr["bytes_h2d"] == int(fp[pf].sum()), (s, r)
            if transfer:
                mo = oms[r].apply(rec[lo:hi], pf - lo, ev - lo)
                assert hdr["bytes_d2h"] == mo["bytes_d2h"], (s, r)
                d2h, h2d = pl.descriptors(hdr)
                assert np.array_equal(h2d[:, 1], mo["h2d_page"]) and np.array_equal(h2d[:, 0], mo["h2d_host"]), (s, r)
                assert np.array_equal(d2h[:, 1], mo["d2h_page"]), (s, r)
        res = p["resident"]
    paths = [pl.list_paths() for pl in ranks]
    for pl in ranks:
        pl.close()
    if expect_paths is not None:
        assert all((f > 0) == (expect_paths == "fast") or (sl > 0) == (expect_paths == "slow") for f, sl in paths), paths
    return paths


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_world_c4_shaped(G):
    """C4-shaped trace (independent agents, C3 footprints, budget 25%), uneven shards."""
    n = 240_000
    w = tg.config_c4(seed=7, steps=10, n=n)
    rng = np.random.default_rng(G)
    inner = np.sort(rng.choice(np.arange(1000, n - 1000), G - 1, replace=False)) if G > 1 else []
    cuts = [0, *[int(x) for x in inner], n]
    paths = run_world(w, cuts)
    assert all(f > 0 for f, _ in paths), paths  # the fast list placement ran


def test_world_tie_group_cut_in_a_later_rank():
    """All agents at one distance: the id-order tie prefix crosses rank 0 entirely and stops
    inside rank 2's shard (the lower ranks' tie bytes come from their published histograms)."""
    n = 60_000
    rng = np.random.default_rng(3)
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    agents = [dict(d=5, fp=int(fp[i])) for i in range(n)]
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    rec = rec_of(agents)[None]
    cuts = [0, 15_000, 31_000, 47_000, n]
    for stop in (31_000 + 17, 31_000 + 5_000, 47_000 - 1):  # the cut falls inside rank 2
        budget = int(fp[:stop].sum())
        w = tg.Workload("ties", n, np.array([0]), rec, None, blocks, budget, np.full(3, 9.0, np.float32))
        run_world(w, cuts)


def test_world_multilevel_select_two_barrier_lists():
    """Distances spread over 1..10^6 ticks with theta = inf (multi-valued buckets everywhere):
    select levels 2-3 over the world's histograms and the two-barrier list path per rank."""
    n = 50_000
    rng = np.random.default_rng(9)
    fp = rng.choice([1, 2], n) * tg.PAGE_BYTES
    recs = []
    for t in range(3):
        d = rng.integers(1, 10 ** 6, n)
        recs.append(rec_of([dict(d=int(d[i]), fp=int(fp[i])) for i in range(n)]))
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    w = tg.Workload("spread", n, np.zeros(3, np.int64), np.stack(recs), None, blocks, int(fp.sum() * 0.3),
                    np.full(3, np.inf, np.float32))
    paths = run_world(w, [0, 20_000, n])
    assert all(sl > 0 for _, sl in paths), paths


def test_world_physical_transfers():
    """C2-mini with physical page copies: each rank assigns and moves the pages of its shard."""
    w = tg.config_c2(seed=2, steps=12, n=3001, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    run_world(w, [0, 1400, 3001], transfer=True)
