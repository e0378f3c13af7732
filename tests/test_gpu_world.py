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


def run_world_tp(w, cuts, content_pages=48):
    """TP-sliced world (SCALESIM_F_TP_SLICED, R16): every rank plans its shard (lists ==
    oracle restricted to the shard), holds the world's merged lists (== the world-1 oracle
    lists), assigns the pages of the whole plan exactly as the world-1 oracle page pool does
    (descriptors and page table), and its arena slot of a loaded page holds its slice of the
    page's host bytes."""
    import torch
    from gpu_harness import fill_pattern
    from paper_2601_21473_b200.planner import Planner, step_group
    G = len(cuts) - 1
    stream = torch.cuda.Stream()
    b = w.blocks
    host = torch.empty(int(b.host_bytes), dtype=torch.uint8, pin_memory=True)
    fill_pattern(host)
    pages = max((w.budget + w.page_bytes - 1) // w.page_bytes, 1)
    su = w.page_bytes // G
    ranks = [Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                     hop_scale=w.hop_scale, transfer=True, page_bytes=w.page_bytes, host_arena=host,
                     dev_bytes=pages * su, shard=(cuts[r], cuts[r + 1]), rank=r, world=G, loopback=True,
                     tp_sliced=True, stream=stream, keep_dist=False) for r in range(G)]
    assert all(pl.fused for pl in ranks)
    om = oracle.OracleMem(b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.page_bytes, pages)
    page_first = np.concatenate([[0], np.cumsum(b.blk_size.astype(np.int64) // w.page_bytes)])
    page_host = np.zeros(int(page_first[-1]), np.int64)  # host offset of every block page
    for blk in range(len(b.blk_size)):
        q0, q1 = int(page_first[blk]), int(page_first[blk + 1])
        page_host[q0:q1] = int(b.blk_host_off[blk]) + np.arange(q1 - q0) * w.page_bytes
    res = np.zeros(w.n, np.uint8)
    rng = np.random.default_rng(0)
    fp = None
    newer = set()  # (slot, rank) written on the device since its last load: newer than the host
    n_wb_checked = 0
    for s in range(w.steps):
        rec = w.rec[s]
        # simulated KV / history writes of dirty resident agents: every rank stamps its slice of
        # their non-LoRA pages; a written-back page must carry each rank's stamp in its slice
        stamped = {}
        pt0 = om.page_table()
        dirty = np.nonzero(((rec[:, 2] >> 4) & 1).astype(bool) & res.astype(bool))[0]
        for a in rng.permutation(dirty)[:6]:
            for blk in range(int(b.blk_ptr[a]), int(b.blk_ptr[a + 1])):
                if b.blk_kind[blk] == tg.KIND_LORA:
                    continue
                for q in range(int(page_first[blk]), int(page_first[blk + 1])):
                    slot = int(pt0[q])
                    for r, pl in enumerate(ranks):
                        mark = np.array([0x7A000000 + s, slot, r, q], np.uint32)
                        pl.dev_arena[slot * su: slot * su + 16].copy_(torch.from_numpy(mark.view(np.uint8)))
                        stamped[(slot, r)] = mark
                        newer.add((slot, r))
        torch.cuda.synchronize()
        for r, pl in enumerate(ranks):
            pl.set_records(rec[cuts[r]:cuts[r + 1]])
        step_group(ranks, int(w.now[s]))
        d, _ = oracle.score(rec, None, int(w.now[s]), w.hop_scale)
        p = oracle.plan(rec, d, res, w.theta, w.budget)
        mo = om.apply(rec, p["prefetch"], p["evict"])
        pt = om.page_table()
        fp = rec[:, 1].astype(np.int64)
        for r, pl in enumerate(ranks):
            lo, hi = cuts[r], cuts[r + 1]
            hdr = pl.sync()
            pf, ev = pl.lists(hdr)
            assert np.array_equal(pf, p["prefetch"][(p["prefetch"] >= lo) & (p["prefetch"] < hi)]), (s, r)
            assert np.array_equal(ev, p["evict"][(p["evict"] >= lo) & (p["evict"] < hi)]), (s, r)
            assert hdr["bytes_h2d"] == int(fp[pf].sum()), (s, r)
            gpf, gev, gh = pl.world_lists()
            assert np.array_equal(gpf, p["prefetch"]) and np.array_equal(gev, p["evict"]), (s, r)
            assert gh["bytes_d2h"] == mo["bytes_d2h"] and gh["status"] == 0, (s, r, gh)
            assert hdr["n_d2h"] == len(mo["d2h_page"]) and hdr["n_h2d"] == len(mo["h2d_page"]), (s, r)
            d2h, h2d = pl.descriptors(hdr)
            assert np.array_equal(h2d[:, 0], mo["h2d_host"]) and np.array_equal(h2d[:, 1], mo["h2d_page"]), (s, r)
            assert np.array_equal(d2h[:, 0], mo["d2h_host"]) and np.array_equal(d2h[:, 1], mo["d2h_page"]), (s, r)
            assert np.array_equal(pl.page_table(), pt), (s, r)
            for k in range(len(d2h)):  # written-back pages: this rank's slice carries its stamp
                ho, slot = int(d2h[k, 0]), int(d2h[k, 1])
                if (slot, r) in stamped:
                    got = host[ho + r * su: ho + r * su + 16].numpy().view(np.uint32)
                    assert np.array_equal(got, stamped[(slot, r)]), (s, r, k, got, stamped[(slot, r)])
                    n_wb_checked += 1
            # content: the rank's slot of a resident page holds slice r of the page's host bytes
            held = np.nonzero(pt != 0xFFFFFFFF)[0]
            for q in rng.permutation(held)[:content_pages]:
                slot, ho = int(pt[q]), int(page_host[q]) + r * su
                if (slot, r) in newer:  # (written on the device since its load: newer than the host)
                    continue
                got = pl.dev_arena[slot * su:(slot + 1) * su].cpu()
                assert torch.equal(got, host[ho:ho + su]), (s, r, int(q), slot)
        res = p["resident"]
        newer -= {(int(x), r) for x in mo["h2d_page"] for r in range(G)}  # (reloaded from the host)
    assert n_wb_checked > 0  # (some stamped slices were written back and checked)
    for pl in ranks:
        pl.close()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_world_tp_sliced_transfers(G):
    """§8(e) step 4 / R16: TP-sliced page transfers of a loopback world (C2-mini, 64 KiB pages:
    32 / 16 / 8 KiB slices, the last below the 16 KB bulk-copy chunk)."""
    w = tg.config_c2(seed=4, steps=10, n=3001, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    assert w.page_bytes == 65536
    cuts = [round(w.n * r / G) for r in range(G + 1)]
    run_world_tp(w, cuts)


def shard_kin(w, s, lo, hi):
    """Rank [lo, hi)'s records of step s with its own kinematics array (the interaction agents of
    its shard, kinematics index rebased) -- the per-rank input of a loopback world."""
    rec = w.rec[s, lo:hi].copy()
    cls = (rec[:, 2] >> 2) & 3
    idx = rec[cls == 1, 3].astype(np.int64)
    if len(idx) == 0:
        return rec, np.zeros((1, 4), np.float32)
    base = int(idx.min())
    assert np.array_equal(np.sort(idx), np.arange(base, base + len(idx)))  # (contiguous in C3)
    rec[cls == 1, 3] = (idx - base).astype(np.uint32)
    return rec, np.ascontiguousarray(w.kin[s, base:base + len(idx)])


@pytest.mark.parametrize("cuts", [[0, 50_000, 100_000], [0, 40_000, 52_000, 100_000]])
def test_world_interaction_kin_allgather(cuts):
    """§8(e) kin all-gather: C3 (three classes) sharded so that every rank holds interaction
    agents; each rank's pair scan sees the world's participants, plan(world) == oracle."""
    import torch
    from paper_2601_21473_b200.planner import Planner, step_group
    w = tg.config_c3(seed=2, steps=3, n=100_000)
    G = len(cuts) - 1
    stream = torch.cuda.Stream()
    ranks = []
    for r in range(G):
        lo, hi = cuts[r], cuts[r + 1]
        bp, bs, bo, bk = shard_blocks(w.blocks, lo, hi)
        _, kin0 = shard_kin(w, 0, lo, hi)
        ranks.append(Planner(w.n, bp, bs, bo, bk, w.budget, w.theta, hop_scale=w.hop_scale, n_kin=len(kin0),
                             transfer=False, shard=(lo, hi), rank=r, world=G, loopback=True, stream=stream,
                             keep_dist=False))
        assert ranks[-1].fused
    res = np.zeros(w.n, np.uint8)
    for s in range(w.steps):
        for r, pl in enumerate(ranks):
            rr, kk = shard_kin(w, s, cuts[r], cuts[r + 1])
            pl.set_records(rr, kk)
        step_group(ranks, int(w.now[s]))
        d, _ = oracle.score(w.rec[s], w.kin[s], int(w.now[s]), w.hop_scale)
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        for r, pl in enumerate(ranks):
            lo, hi = cuts[r], cuts[r + 1]
            hdr = pl.sync()
            pf, ev = pl.lists(hdr)
            assert np.array_equal(pf, p["prefetch"][(p["prefetch"] >= lo) & (p["prefetch"] < hi)]), (s, r)
            assert np.array_equal(ev, p["evict"][(p["evict"] >= lo) & (p["evict"] < hi)]), (s, r)
            assert np.array_equal(pl.resident(), p["resident"][lo:hi]), (s, r)
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"], (s, r)
            assert hdr["kept_bytes"] == p["kept_bytes"] and hdr["n_eligible"] == p["n_eligible"], (s, r)
        res = p["resident"]
    for pl in ranks:
        pl.close()


def run_world_threads(w, cuts, transfer=False):
    """The multi-kernel world > 1 path (the NCCL path's launches and collectives) with the
    SCALESIM_F_THREADS exchange: one context per rank on this device, each stepped by its own
    host thread; plan(world) == oracle restricted to each shard, bit for bit."""
    import threading
    import torch
    from gpu_harness import fill_pattern
    from paper_2601_21473_b200.planner import Planner
    G = len(cuts) - 1
    gid = bytes([7, G]) + bytes(126)
    host = None
    if transfer:
        host = torch.empty(int(w.blocks.host_bytes), dtype=torch.uint8, pin_memory=True)
        fill_pattern(host)
    ranks, oms = [], []
    pages = max((w.budget + w.page_bytes - 1) // w.page_bytes, 1)
    for r in range(G):
        lo, hi = cuts[r], cuts[r + 1]
        bp, bs, bo, bk = shard_blocks(w.blocks, lo, hi)
        ranks.append(Planner(w.n, bp, bs, bo, bk, w.budget, w.theta, hop_scale=w.hop_scale, transfer=transfer,
                             page_bytes=w.page_bytes, host_arena=host, dev_bytes=pages * w.page_bytes,
                             shard=(lo, hi), rank=r, world=G, nccl_id=gid, threads=True, keep_dist=False))
        assert not ranks[-1].fused  # (the multi-kernel path)
        if transfer:
            oms.append(oracle.OracleMem(bp, bs, bo, bk, w.page_bytes, pages))
    res = np.zeros(w.n, np.uint8)
    for s in range(w.steps):
        rec = w.rec[s]
        errs = []

        def run(r):
            try:
                ranks[r].set_records(rec[cuts[r]:cuts[r + 1]])
                ranks[r].step(int(w.now[s]))
            except Exception as e:  # noqa: BLE001
                errs.append((r, e))
        th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not errs and not any(t.is_alive() for t in th), errs
        d, _ = oracle.score(rec, None, int(w.now[s]), w.hop_scale)
        p = oracle.plan(rec, d, res, w.theta, w.budget)
        fp = rec[:, 1].astype(np.int64)
        for r, pl in enumerate(ranks):
            lo, hi = cuts[r], cuts[r + 1]
            hdr = pl.sync()
            pf, ev = pl.lists(hdr)
            assert np.array_equal(pf, p["prefetch"][(p["prefetch"] >= lo) & (p["prefetch"] < hi)]), (s, r)
            assert np.array_equal(ev, p["evict"][(p["evict"] >= lo) & (p["evict"] < hi)]), (s, r)
            assert np.array_equal(pl.resident(), p["resident"][lo:hi]), (s, r)
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"], (s, r)
            assert hdr["kept_bytes"] == p["kept_bytes"], (s, r, hdr["kept_bytes"], p["kept_bytes"])
            assert hdr["bytes_h2d"] == int(fp[pf].sum()), (s, r)
            if transfer:
                mo = oms[r].apply(rec[lo:hi], pf - lo, ev - lo)
                assert hdr["bytes_d2h"] == mo["bytes_d2h"], (s, r)
                d2h, h2d = pl.descriptors(hdr)
                assert np.array_equal(h2d[:, 1], mo["h2d_page"]) and np.array_equal(h2d[:, 0], mo["h2d_host"]), (s, r)
        res = p["resident"]
    for pl in ranks:
        pl.close()


@pytest.mark.parametrize("G", [2, 3, 4])
def test_world_threads_multikernel(G):
    """The NCCL path's plan sequence (7 collectives per step) over the thread exchange, C4-shaped."""
    n = 120_000
    w = tg.config_c4(seed=11, steps=6, n=n)
    cuts = [round(n * r / G) + (0 if r in (0, G) else 137 * r) for r in range(G + 1)]
    run_world_threads(w, cuts)


def test_world_threads_tie_cut_and_transfers():
    """Tie cut inside rank 1 (id-order prefix across ranks through the gathered tie bytes) and
    per-rank physical transfers on the multi-kernel world path."""
    n = 30_000
    rng = np.random.default_rng(5)
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    rec = rec_of([dict(d=5, fp=int(fp[i])) for i in range(n)])[None]
    budget = int(fp[:12_345].sum())
    w = tg.Workload("ties", n, np.array([0]), rec, None, blocks, budget, np.full(3, 9.0, np.float32))
    run_world_threads(w, [0, 10_000, 20_000, n])
    w2 = tg.config_c2(seed=3, steps=8, n=3001, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    run_world_threads(w2, [0, 1500, 3001], transfer=True)


def test_world_threads_rejects_non_contiguous_shards():
    """the tie prefix over lower ranks assumes contiguous shards in rank order; a world
    whose shards leave a gap fails its first collective with SCALESIM_E_INVALID on every rank."""
    import threading
    from paper_2601_21473_b200 import _lib as L
    from paper_2601_21473_b200.planner import Planner
    n = 4000
    w = tg.config_c4(seed=2, steps=1, n=n)
    cuts = [(0, 1500), (1700, n)]
    gid = bytes([9, 2]) + bytes(126)
    ranks = []
    for r, (lo, hi) in enumerate(cuts):
        bp, bs, bo, bk = shard_blocks(w.blocks, lo, hi)
        ranks.append(Planner(n, bp, bs, bo, bk, w.budget, w.theta, transfer=False, shard=(lo, hi), rank=r, world=2,
                             nccl_id=gid, threads=True, keep_dist=False))
    codes = {}

    def run(r):
        lo, hi = cuts[r]
        ranks[r].set_records(w.rec[0][lo:hi])
        try:
            ranks[r].step(int(w.now[0]))
            codes[r] = 0
        except L.ScaleSimError as e:
            codes[r] = e.status
    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert codes == {0: L.E_INVALID, 1: L.E_INVALID}, codes
    for pl in ranks:
        pl.close()
