"""GPU parity: the CUDA planner (through the C ABI) against the CPU oracle, element by
element, on seeded workloads of every BASELINE config shape."""
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


PATHS = [pytest.param(False, id="fused"), pytest.param(True, id="multikernel")]


@pytest.mark.parametrize("mk", PATHS)
def test_c1_all_variants(mk):
    from gpu_harness import run_parity
    for variant in ("ind", "int", "diff", "diff-star"):
        for th in (0.0, 3.0, np.inf):
            for seed in (1, 2, 3):
                w = tg.config_c1(seed=seed, theta=(th, th, th), variant=variant)
                run_parity(w, multi_kernel=mk)


@pytest.mark.parametrize("mk", PATHS)
def test_c2_mini_physical_transfer(mk):
    from gpu_harness import run_parity
    w = tg.config_c2(seed=2, steps=40, n=3001, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    out = run_parity(w, multi_kernel=mk)
    assert sum(o["n_evict"] for o in out) > 0


@pytest.mark.parametrize("mk", PATHS)
def test_c3_mini_all_classes(mk):
    from gpu_harness import run_parity
    w = tg.config_c3(seed=1, steps=6, n=9001, budget=int(9001 * 3.41e6 * 0.235), host_bytes=4 << 30)
    run_parity(w, stamp_writes=False, multi_kernel=mk)


def test_c2_full_size():
    """BASELINE configs[1]: 10k agents, rank-16 7B LoRA + 917,504 B KV pages, budget 25%."""
    from gpu_harness import run_parity
    w = tg.config_c2(seed=1, steps=24, host_bytes=16 << 30)
    run_parity(w, stamp_writes=False, content_pages=16)


def test_c3_full_size():
    """BASELINE configs[2]: 100k agents, three classes, 80 GB budget (2 steps: the oracle's
    O(n^2) interaction scan takes ~10 s per step)."""
    from gpu_harness import run_parity
    w = tg.config_c3(seed=1, steps=2, host_bytes=8 << 30)
    run_parity(w, stamp_writes=False, content_pages=16)


@pytest.mark.parametrize("mk,keep,excl", [pytest.param(False, True, False, id="fused"),
                                          pytest.param(False, False, True, id="fused-nokeep-exclusive-bench"),
                                          pytest.param(True, True, False, id="multikernel")])
def test_c4_full_size_logical(mk, keep, excl):
    """BASELINE configs[3] at G=1: 1M agents, logical sizes (no arena).  `fused-nokeep-
    exclusive-bench` is exactly bench.py's headline configuration (same generator, seed and
    size; keep_dist off: the fused kernel's fast P1 variant; SCALESIM_F_EXCLUSIVE: the launch
    without the cooperative attribute)."""
    from gpu_harness import run_parity
    w = tg.config_c4(seed=1, steps=6 if mk else 24)
    out = run_parity(w, transfer=False, multi_kernel=mk, keep_dist=keep, exclusive=excl)
    if not mk:  # integer distances: most steps place their lists without the second barrier
        fast, slow = out[-1]["paths"]
        assert fast + slow == 24 and fast >= 12, (fast, slow)


@pytest.mark.parametrize("mk", PATHS)
def test_edge_cases(mk):
    from gpu_harness import run_parity as _rp

    def run_parity(w, **kw):
        return _rp(w, multi_kernel=mk, **kw)
    PG = tg.PAGE_BYTES

    def wl(agents, budget, theta=(4.0, 4.0, 4.0), kin=None, now=0, resident=None):
        n = len(agents)
        for a in agents:
            a.setdefault("fp", PG)
        blocks = tg.make_blocks([[tg.KIND_KV] if a["fp"] else [] for a in agents],
                                [[a["fp"]] if a["fp"] else [] for a in agents])
        rec = rec_of(agents, now)[None]
        k = None if kin is None else np.asarray(kin, np.float32)[None]
        return tg.Workload("edge", n, np.array([now]), rec, k, blocks, budget, np.asarray(theta, np.float32))

    # single agent, fits / does not fit
    run_parity(wl([dict(d=1)], PG))
    run_parity(wl([dict(d=1)], PG - 1))
    # ragged word (33 agents), everything fits
    run_parity(wl([dict(d=i % 5) for i in range(33)], 40 * PG))
    # budget 0 with active agents -> INSUFFICIENT
    run_parity(wl([dict(phase=tg.PH_GENERATING), dict(d=2)], 0))
    # theta 0 and inf, idle agents, unreachable diffusion, zero-footprint agents
    ag = [dict(d=3), dict(phase=tg.PH_IDLE), dict(cls=tg.CL_DIFF, hop=tg.UNREACHABLE), dict(d=1, fp=0),
          dict(cls=tg.CL_DIFF, hop=2), dict(phase=tg.PH_WAITING)]
    for th in (0.0, np.inf):
        run_parity(wl([dict(a) for a in ag], 3 * PG, theta=(th, th, th)))
    # malformed records: class 3, kin index out of range, non-finite kinematics
    ag = [dict(cls=3, d=2), dict(cls=tg.CL_INT, d=5, kin=9), dict(cls=tg.CL_INT, d=5, kin=0),
          dict(cls=tg.CL_INT, d=5, kin=1)]
    run_parity(wl(ag, 10 * PG, kin=[[0, 0, np.nan, 0], [1, 0, -1, 0]]))
    # resident at init, then evicted
    w = wl([dict(d=9), dict(d=1), dict(phase=tg.PH_GENERATING)], 2 * PG)
    run_parity(w, resident_init=np.array([1, 1, 0], np.uint8))


@pytest.mark.parametrize("mk", PATHS)
def test_large_tie_group_spans_tiles(mk):
    """Heavy integer ties: 20,000 agents at the same distance, budget cutting inside the tie
    group across several 2048-agent tiles (id-order prefix, R1/R3)."""
    from gpu_harness import run_parity as _rp

    def run_parity(w, **kw):
        return _rp(w, multi_kernel=mk, **kw)
    n = 20000
    rng = np.random.default_rng(3)
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    agents = [dict(d=5, fp=int(fp[i])) for i in range(n)]
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    rec = rec_of(agents)[None]
    budget = int(fp.sum() * 0.37)
    w = tg.Workload("ties", n, np.array([0]), rec, None, blocks, budget, np.full(3, 9.0, np.float32))
    run_parity(w)
    run_parity(w, transfer=False)
    run_parity(w, transfer=False, keep_dist=False)


def test_call_order_and_host_step():
    from paper_2601_21473_b200 import _lib as L
    from gpu_harness import make_planner
    w = tg.config_c2(seed=4, steps=3, n=500, lora=2 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    pl = make_planner(w, transfer=True)
    with pytest.raises(L.ScaleSimError) as e:
        pl.plan()
    assert e.value.status == L.E_ORDER
    pl.set_records(w.rec[0])
    pl.score(int(w.now[0]))
    pl.plan()
    pl.transfer()
    with pytest.raises(L.ScaleSimError):
        pl.transfer()
    hdr = pl.sync()
    # the end-to-end host entry point gives the same plan as the device one
    pl2 = make_planner(w, transfer=True)
    pf = np.zeros(w.n, np.uint32)
    ev = np.zeros(w.n, np.uint32)
    h2 = pl2.step_host(int(w.now[0]), np.ascontiguousarray(w.rec[0]), None, pf, ev)
    pf1, ev1 = pl.lists(hdr)
    assert h2["n_prefetch"] == hdr["n_prefetch"] and np.array_equal(pf[:h2["n_prefetch"]], pf1)
    assert h2["cut_bits"] == hdr["cut_bits"] and h2["bytes_h2d"] == hdr["bytes_h2d"]
    pl.close()
    pl2.close()


@pytest.mark.parametrize("exclusive", [False, True])
def test_pipelined_host_steps_c4_shape(exclusive):
    """scalesim_stage_host + scalesim_step_host back to back (step t+1's records cross the link
    while step t plans, keep_dist=False as benched): every step's header and lists equal the
    oracle's; the staged buffers rotate, a fourth outstanding stage is refused."""
    import torch
    from paper_2601_21473_b200 import _lib as L
    from gpu_harness import make_planner
    w = tg.config_c4(seed=5, steps=7, n=300_000)
    pl = make_planner(w, transfer=False, keep_dist=False, exclusive=exclusive)
    recs = [torch.from_numpy(np.ascontiguousarray(w.rec[s])).pin_memory().numpy() for s in range(w.steps)]
    pf = np.zeros(w.n, np.uint32)
    ev = np.zeros(w.n, np.uint32)
    res = np.zeros(w.n, np.uint8)
    pl.stage_host(recs[0])
    for s in range(w.steps):
        if s + 1 < w.steps and s != 1:  # (recs[2] was staged at s == 0)
            pl.stage_host(recs[s + 1])
            if s == 0:  # three staged steps at most
                pl.stage_host(recs[2])
                with pytest.raises(L.ScaleSimError) as e:
                    pl.stage_host(recs[3])
                assert e.value.status == L.E_ORDER
        h = pl.step_host(int(w.now[s]), recs[s], None, pf, ev)
        d_or, _ = oracle.score(w.rec[s], None, int(w.now[s]), w.hop_scale)
        p = oracle.plan(w.rec[s], d_or, res, w.theta, w.budget)
        assert h["cut_bits"] == p["cut_bits"] and h["cut_rem"] == p["cut_rem"], s
        assert h["kept_bytes"] == p["kept_bytes"] and h["bytes_h2d"] == p["bytes_h2d"], s
        assert h["n_prefetch"] == len(p["prefetch"]) and h["n_evict"] == len(p["evict"]), s
        assert np.array_equal(pf[:h["n_prefetch"]], p["prefetch"]), s
        assert np.array_equal(ev[:h["n_evict"]], p["evict"]), s
        res = p["resident"].astype(np.uint8)
    pl.close()


def test_pipelined_host_steps_with_kinematics():
    """scalesim_stage_host with kinematics (C3-mini: interaction agents, n_kin > 0): the staged
    records AND kinematics reach the plan of their own step (the pair scan reads the staged
    kinematics), every step's header and lists equal the oracle's."""
    import torch
    from gpu_harness import make_planner
    w = tg.config_c3(seed=2, steps=5, n=9001, budget=int(9001 * 3.41e6 * 0.235), host_bytes=4 << 30)
    assert w.n_kin > 0
    pl = make_planner(w, transfer=False)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    recs = [pin(w.rec[s]) for s in range(w.steps)]
    kins = [pin(w.kin[s]) for s in range(w.steps)]
    pf = np.zeros(w.n, np.uint32)
    ev = np.zeros(w.n, np.uint32)
    res = np.zeros(w.n, np.uint8)
    pl.stage_host(recs[0], kins[0])
    for s in range(w.steps):
        if s + 1 < w.steps:
            pl.stage_host(recs[s + 1], kins[s + 1])
        h = pl.step_host(int(w.now[s]), recs[s], kins[s], pf, ev)
        d_or, _ = oracle.score(w.rec[s], w.kin[s], int(w.now[s]), w.hop_scale)
        p = oracle.plan(w.rec[s], d_or, res, w.theta, w.budget)
        _assert_host_plan(h, pf, ev, p, s)
        res = p["resident"].astype(np.uint8)
    pl.close()


def _oracle_step(w, s, res):
    d_or, _ = oracle.score(w.rec[s], None, int(w.now[s]), w.hop_scale)
    return oracle.plan(w.rec[s], d_or, res, w.theta, w.budget)


def _assert_host_plan(h, pf, ev, p, s):
    assert h["cut_bits"] == p["cut_bits"] and h["cut_rem"] == p["cut_rem"], s
    assert h["kept_bytes"] == p["kept_bytes"] and h["bytes_h2d"] == p["bytes_h2d"], s
    assert h["n_prefetch"] == len(p["prefetch"]) and h["n_evict"] == len(p["evict"]), s
    assert np.array_equal(pf[:h["n_prefetch"]], p["prefetch"]), s
    assert np.array_equal(ev[:h["n_evict"]], p["evict"]), s


@pytest.mark.parametrize("exclusive", [False, True])
def test_incremental_host_steps_c4_shape(exclusive):
    """scalesim_stage_updates + scalesim_step_updates (the bench's e2e loop): after one whole
    upload, each step sends only the records that changed; staged one step ahead, plus one
    unstaged step and one step without changes; every plan equals the oracle's on the full
    records.  An id outside the shard is reported (E_BAD_INPUT) and skipped."""
    import torch
    from paper_2601_21473_b200 import _lib as L
    from gpu_harness import make_planner
    w = tg.config_c4(seed=6, steps=8, n=300_000)
    w.rec[5] = w.rec[4]  # a step without changes
    pl = make_planner(w, transfer=False, keep_dist=False, exclusive=exclusive)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    ids, recs = [None], [None]
    for s in range(1, w.steps):
        ch = np.nonzero(np.any(w.rec[s] != w.rec[s - 1], axis=1))[0].astype(np.uint32)
        ids.append(pin(ch))
        recs.append(pin(w.rec[s][ch]))
    assert len(ids[5]) == 0 and 0 < len(ids[1]) < w.n // 5
    pf = np.zeros(w.n, np.uint32)
    ev = np.zeros(w.n, np.uint32)
    res = np.zeros(w.n, np.uint8)
    h = pl.step_host(int(w.now[0]), pin(w.rec[0]), None, pf, ev)
    p = _oracle_step(w, 0, res)
    _assert_host_plan(h, pf, ev, p, 0)
    res = p["resident"].astype(np.uint8)
    pl.stage_updates(ids[1], recs[1])
    for s in range(1, w.steps):
        if s + 1 < w.steps and s != 2:  # step 3 is not staged: its copy is synchronous
            pl.stage_updates(ids[s + 1], recs[s + 1])
        h = pl.step_updates(int(w.now[s]), ids[s], recs[s], pf, ev)
        p = _oracle_step(w, s, res)
        _assert_host_plan(h, pf, ev, p, s)
        res = p["resident"].astype(np.uint8)
    bad = pin(np.array([w.n + 7], np.uint32))
    with pytest.raises(L.ScaleSimError) as e:
        pl.step_updates(int(w.now[w.steps - 1]), bad, pin(w.rec[0][:1]), pf, ev)
    assert e.value.status == L.E_BAD_INPUT
    pl.close()


@pytest.mark.parametrize("n,exclusive", [(300_000, False), (300_000, True), (1_000_000, True)],
                         ids=["300k-coop", "300k-excl", "bench-e2e-c4-1M-excl"])
def test_submitted_incremental_steps_c4_shape(n, exclusive):
    """scalesim_submit_updates / scalesim_collect (three steps in flight: steps t+1, t+2 copy and
    plan while the host collects t; at 1M agents, exclusive, keep_dist off: the bench's e2e configuration):
    every collected plan equals the oracle's on the full records; a third submission and
    step_host with steps pending are refused; an out-of-shard id is reported by the collect of
    its own step only."""
    import torch
    from paper_2601_21473_b200 import _lib as L
    from gpu_harness import make_planner
    w = tg.config_c4(seed=7, steps=7, n=n)
    pl = make_planner(w, transfer=False, keep_dist=False, exclusive=exclusive)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    ids, recs = [None], [None]
    for s in range(1, w.steps):
        ch = np.nonzero(np.any(w.rec[s] != w.rec[s - 1], axis=1))[0].astype(np.uint32)
        ids.append(pin(ch))
        recs.append(pin(w.rec[s][ch]))
    pf = np.zeros(w.n, np.uint32)
    ev = np.zeros(w.n, np.uint32)
    res = np.zeros(w.n, np.uint8)
    rec0 = pin(w.rec[0])
    h = pl.step_host(int(w.now[0]), rec0, None, pf, ev)
    p = _oracle_step(w, 0, res)
    _assert_host_plan(h, pf, ev, p, 0)
    res = p["resident"].astype(np.uint8)
    pl.submit_updates(int(w.now[1]), ids[1], recs[1])
    pl.submit_updates(int(w.now[2]), ids[2], recs[2])
    for s in range(1, w.steps):
        if s + 2 < w.steps:
            pl.submit_updates(int(w.now[s + 2]), ids[s + 2], recs[s + 2])
            if s == 1:  # three steps in flight at most
                with pytest.raises(L.ScaleSimError) as e:
                    pl.submit_updates(int(w.now[s + 3]), ids[s + 3], recs[s + 3])
                assert e.value.status == L.E_ORDER
                with pytest.raises(L.ScaleSimError) as e:
                    pl.step_host(int(w.now[0]), rec0, None, pf, ev)
                assert e.value.status == L.E_ORDER
        h = pl.collect(pf, ev)
        p = _oracle_step(w, s, res)
        _assert_host_plan(h, pf, ev, p, s)
        res = p["resident"].astype(np.uint8)
    with pytest.raises(L.ScaleSimError) as e:
        pl.collect(pf, ev)
    assert e.value.status == L.E_ORDER
    last = w.steps - 1
    bad = pin(np.array([w.n + 3], np.uint32))
    pl.submit_updates(int(w.now[last]), bad, pin(w.rec[last][:1]))
    pl.submit_updates(int(w.now[last]), pin(np.zeros(0, np.uint32)), pin(np.zeros((0, 4), np.uint32)))
    with pytest.raises(L.ScaleSimError) as e:
        pl.collect(pf, ev)
    assert e.value.status == L.E_BAD_INPUT
    h = pl.collect(pf, ev)  # the next step has no bad id (both plan the last records again)
    res = _oracle_step(w, last, res)["resident"].astype(np.uint8)
    p = _oracle_step(w, last, res)
    _assert_host_plan(h, pf, ev, p, last)
    pl.close()


def test_fused_multi_level_select_and_segments():
    """Distances spread over many values (boundary bucket with several distances: select
    levels 2 and 3; evict segments that need the re-sort by full key), fused vs oracle."""
    from gpu_harness import run_parity
    n = 50000
    rng = np.random.default_rng(9)
    d = rng.integers(1, 5000, n)
    fp = rng.choice([1, 2], n) * tg.PAGE_BYTES
    agents = [dict(d=int(d[i]), fp=int(fp[i])) for i in range(n)]
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    rec0 = rec_of(agents)
    # second step: everyone's distance changes (large evict list over many distances)
    agents2 = [dict(d=int(x), fp=int(fp[i])) for i, x in enumerate(rng.integers(1, 5000, n))]
    rec = np.stack([rec0, rec_of(agents2)])
    budget = int(fp.sum() * 0.3)
    w = tg.Workload("spread", n, np.array([0, 0]), rec, None, blocks, budget, np.full(3, np.inf, np.float32))
    run_parity(w, transfer=False)
    run_parity(w, transfer=False, keep_dist=False)  # (staged P1 records, two-barrier list path)
    run_parity(w, transfer=False, multi_kernel=True)
    run_parity(w)


def test_c5_batch_replicas_vs_oracle():
    """BASELINE configs[4] shape: independent replicas x budgets planned by one batched
    launch (scalesim_step_batch); every instance equals its own oracle run."""
    import torch
    from paper_2601_21473_b200.planner import Planner, step_batch
    replicas, budgets, n, steps = 3, (10, 40, 90), 2000, 10
    ws = [tg.config_c5(replica=r, budget_pct=10, steps=steps, n=n) for r in range(replicas)]
    stream = torch.cuda.Stream()
    inst = []
    for r, w in enumerate(ws):
        total = int(w.footprint.sum())
        for pct in budgets:
            b = w.blocks
            budget = total * pct // 100
            pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta,
                         transfer=False, stream=stream)
            assert pl.fused
            inst.append(dict(pl=pl, w=w, budget=budget, res=np.zeros(n, np.uint8)))
    for s in range(steps):
        for it in inst:
            it["pl"].set_records(it["w"].rec[s])
        step_batch([it["pl"] for it in inst], int(ws[0].now[s]))
        for it in inst:
            w = it["w"]
            hdr = it["pl"].sync()
            d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
            p = oracle.plan(w.rec[s], d, it["res"], w.theta, it["budget"])
            pf, ev = it["pl"].lists(hdr)
            assert np.array_equal(pf, p["prefetch"]) and np.array_equal(ev, p["evict"]), s
            assert np.array_equal(it["pl"].resident(), p["resident"])
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"]
            assert hdr["kept_bytes"] == p["kept_bytes"] and hdr["bytes_h2d"] == p["bytes_h2d"]
            it["res"] = p["resident"]
    for it in inst:
        it["pl"].close()


def test_fused_wide_code_segments():
    """Large integer distances (2^17..2^24 ticks: one list bucket spans up to 2^19 distinct
    values) so the list segments need the full radix sort: whole-list changes give long
    segments sorted in global memory, a 3% change gives short ones sorted in shared memory."""
    from gpu_harness import run_parity
    n = 50000
    rng = np.random.default_rng(17)
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    d0 = rng.integers(1 << 17, 1 << 24, n)
    d1 = d0.copy()
    ch = rng.choice(n, n * 3 // 100, replace=False)
    d1[ch] = rng.integers(1 << 17, 1 << 24, len(ch))
    recs = [rec_of([dict(d=int(x), fp=int(fp[i])) for i, x in enumerate(dd)]) for dd in (d0, d1, d0)]
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    w = tg.Workload("wide", n, np.zeros(3, np.int64), np.stack(recs), None, blocks, int(fp.sum() * 0.3),
                    np.full(3, np.inf, np.float32))
    run_parity(w, transfer=False)
    run_parity(w, transfer=False, keep_dist=False)
    run_parity(w, transfer=False, multi_kernel=True)


@pytest.mark.parametrize("keep", [True, False])
def test_remaining_ticks_beyond_2_24(keep):
    """R8 at the GPU: remaining action times from 2^24 up to the largest 32-bit t_next (cast
    round-to-nearest-even, halfway cases included) mixed with small ones; the boundary falls
    among the large values in some steps and among the small ones in others."""
    from gpu_harness import run_parity
    n = 40000
    now = 1000
    rng = np.random.default_rng(29)
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    steps = []
    for s in range(3):
        big = rng.random(n) < (0.2 if s != 1 else 0.7)
        d = np.where(big, rng.integers(1 << 24, 0xFFFFFFFF - now, n), rng.integers(0, 60, n))
        d[:8] = [(1 << 24) + 1, (1 << 24) + 3, (1 << 25) + 2, (1 << 25) + 6, 0xFFFFFFFF - now, 1 << 24, (1 << 24) - 1, 0]
        steps.append(rec_of([dict(d=int(x), fp=int(fp[i])) for i, x in enumerate(d)], now))
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    w = tg.Workload("wide24", n, np.full(3, now, np.int64), np.stack(steps), None, blocks, int(fp.sum() * 0.3),
                    np.full(3, 40.0, np.float32))
    run_parity(w, transfer=False, keep_dist=keep)
    if keep:
        run_parity(w, transfer=False, multi_kernel=True)


@pytest.mark.parametrize("mk", PATHS)
def test_interaction_grid_pruning_exact(mk):
    """a1' with the spatial grid (>= 2048 participants): clusters far denser than the grid,
    agents on cell boundaries and at identical positions, stationary agents, fast agents,
    D_action from 0 to 10^6 ticks; distances bit-identical to the oracle's all-pairs scan."""
    from gpu_harness import run_parity
    rng = np.random.default_rng(21)
    n = 6000
    pos = rng.uniform(0, 3000, (n, 2))
    pos[:1500] = rng.normal(1500, 3.0, (1500, 2))               # one dense cluster
    pos[1500:1700] = np.round(pos[1500:1700] / 50.0) * 50.0      # grid-aligned coordinates
    pos[1700:1710] = pos[1700]                                   # identical positions
    vel = rng.normal(0, 1, (n, 2))
    vel[2000:2500] = 0.0                                         # stationary
    vel[2500:2600] *= 40.0                                       # fast
    kin = np.concatenate([pos, vel], axis=1).astype(np.float32)
    d_action = rng.integers(0, 60, n)
    d_action[:100] = 0
    d_action[100:200] = 10 ** 6
    steps = []
    for s in range(2):
        k = kin.copy()
        k[:, :2] += s * k[:, 2:]
        agents = [dict(cls=tg.CL_INT, d=int(d_action[i]), kin=i, fp=tg.PAGE_BYTES) for i in range(n)]
        for i in rng.choice(n, 300, replace=False):
            agents[i]["phase"] = tg.PH_GENERATING
        steps.append((rec_of(agents), k))
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[tg.PAGE_BYTES]] * n)
    w = tg.Workload("grid", n, np.zeros(2, np.int64), np.stack([r for r, _ in steps]),
                    np.stack([k for _, k in steps]), blocks, n * tg.PAGE_BYTES // 3, np.full(3, 30.0, np.float32))
    run_parity(w, transfer=False, multi_kernel=mk)


@pytest.mark.parametrize("mk", PATHS)
def test_tie_cut_word_boundaries_and_writebacks(mk):
    """The budget cut lands exactly on word / tile boundaries of the d == D* tie group, with
    zero-size tie agents right at the cut (kept: inclusive prefix <= rem), and dirty resident
    agents both beyond D* and inside the tie group past the cut (write-back bytes, R13)."""
    from gpu_harness import run_parity as _rp
    rng = np.random.default_rng(11)
    n = 70000  # several fused tiles (~473 agents per CTA at 148 CTAs) and ragged words
    PG = tg.PAGE_BYTES
    d = np.where(rng.random(n) < 0.6, 5, rng.integers(1, 40, n))
    fp = rng.choice([0, 1, 2], n, p=[0.1, 0.6, 0.3]) * PG
    dirty = (rng.random(n) < 0.5).astype(int)
    agents = [dict(d=int(d[i]), fp=int(fp[i]), dirty=int(dirty[i])) for i in range(n)]
    blocks = tg.make_blocks([[tg.KIND_KV] if f else [] for f in fp], [[int(f)] if f else [] for f in fp])
    rec = rec_of(agents)[None]
    below = int(fp[(d < 5)].sum())
    tie_ids = np.nonzero(d == 5)[0]
    csum = np.cumsum(fp[tie_ids])
    resident = (rng.random(n) < 0.5).astype(np.uint8)
    for j in (31, 32 * 40 - 1, len(tie_ids) // 2):  # cut after the j-th tie agent (in id order)
        budget = below + int(csum[j])
        w = tg.Workload("tiecut", n, np.array([0]), rec, None, blocks, budget, np.full(3, 50.0, np.float32))
        _rp(w, transfer=False, multi_kernel=mk, resident_init=resident)
        if not mk:  # the bench's fast P1 variant (no distance copy)
            _rp(w, transfer=False, resident_init=resident, keep_dist=False)


def test_batch_single_cta_instances():
    """scalesim_step_batch with >= 75 instances gives each instance one CTA (the C5 launch
    shape on one GPU): its lists come from the single-CTA paths (per-segment counting when
    every multi-valued list bucket holds <= 128 members, else a radix sort: the `wide`
    workload), or from the slot path when a list exceeds 3/4 of the tile (theta = inf,
    budget 90%)."""
    import torch
    from paper_2601_21473_b200.planner import Planner, step_batch
    n, steps, k = 1500, 6, 80
    ws = [tg.config_c5(replica=r, budget_pct=10, steps=steps, n=n) for r in range(7)]
    # one workload whose distances share one list bucket ([16, 32): several values per bucket,
    # far more than 128 members): the radix-sort fallback
    rng = np.random.default_rng(5)
    fpw = rng.choice([1, 2], n) * tg.PAGE_BYTES
    now = np.asarray(ws[0].now, np.int64)  # (one `now` per batched step for every instance)
    recw = np.stack([rec_of([dict(d=int(rng.integers(16, 20)), fp=int(fpw[a]), dirty=int(rng.integers(0, 2)))
                             for a in range(n)], now=int(now[t])) for t in range(steps)])
    blw = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fpw])
    wide = tg.Workload("wide", n, now, recw, None, blw, int(fpw.sum()) // 2, np.full(3, 50.0, np.float32))
    ws.append(wide)
    stream = torch.cuda.Stream()
    inst = []
    for i in range(k):
        w = ws[i % 8]
        pct = 90 if i >= k - 2 else (40 if i >= k - 4 else 10 * (1 + i % 9))
        theta = np.full(3, np.inf, np.float32) if i >= k - 4 else w.theta
        b = w.blocks
        budget = int(b.blk_size.astype(np.int64).sum()) * pct // 100
        pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, theta, transfer=False,
                     stream=stream)
        inst.append(dict(pl=pl, w=w, budget=budget, theta=theta, res=np.zeros(n, np.uint8)))
    for s in range(steps):
        for it in inst:
            it["pl"].set_records(it["w"].rec[s])
        step_batch([it["pl"] for it in inst], int(ws[0].now[s]))
        for i, it in enumerate(inst):
            w = it["w"]
            hdr = it["pl"].sync()
            d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
            p = oracle.plan(w.rec[s], d, it["res"], it["theta"], it["budget"])
            pf, ev = it["pl"].lists(hdr)
            assert np.array_equal(pf, p["prefetch"]) and np.array_equal(ev, p["evict"]), (s, i)
            assert np.array_equal(it["pl"].resident(), p["resident"]), (s, i)
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["kept_bytes"] == p["kept_bytes"], (s, i)
            assert hdr["bytes_h2d"] == p["bytes_h2d"], (s, i)
            dirty = ((w.rec[s][:, 2] >> 4) & 1).astype(bool)  # R13 write-back bytes of dirty evicted agents
            bl = w.blocks
            wb = sum(int(bl.blk_size[int(bl.blk_ptr[a]):int(bl.blk_ptr[a + 1])][
                bl.blk_kind[int(bl.blk_ptr[a]):int(bl.blk_ptr[a + 1])] != tg.KIND_LORA].astype(np.int64).sum())
                for a in p["evict"] if dirty[a])
            assert hdr["bytes_d2h"] == wb, (s, i)
            it["res"] = p["resident"]
    for it in inst:
        it["pl"].close()
