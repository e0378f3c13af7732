"""GPU parity on the exact configurations bench.py times (VERDICT r1 "weak" #1), plus stream
ordering of back-to-back physical transfers.

- C5 at the bench's shape: 64 replicas x 9 budgets (10..90%) of the C2 shape, 10k agents
  each = 576 instances on one GPU, plan-only, keep_dist off, all stepped by
  scalesim_step_batch on one stream (bench.py c5_leg): every instance against its own oracle
  run, every step.
- Back-to-back physical transfers: scalesim_step called for several steps without any host
  synchronisation, with a device arena exactly as large as the budget (recycled pages are
  reused by the very next step); host copies of written-back pages must carry the device
  contents they had when they were evicted.
(The C4 headline configuration is tests/test_gpu_parity.py::test_c4_full_size_logical
[fused-nokeep-bench].)
"""
import numpy as np
import pytest

import oracle
import tracegen as tg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


def test_c5_bench_shape_576_instances():
    import torch
    from paper_2601_21473_b200.planner import Planner, step_batch
    replicas, budgets, steps = 64, tuple(range(10, 100, 10)), 16  # bench.py c5_leg defaults (warm 8 + timed 8)
    traces = {r: tg.config_c5(replica=r, budget_pct=10, seed_base=100, steps=steps) for r in range(replicas)}
    stream = torch.cuda.Stream()
    inst = []
    for r in range(replicas):
        w = traces[r]
        b = w.blocks
        for pct in budgets:
            budget = int(w.footprint.sum()) * pct // 100
            pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, budget, w.theta, transfer=False,
                         stream=stream, keep_dist=False)
            assert pl.fused
            inst.append(dict(pl=pl, w=w, budget=budget, res=np.zeros(w.n, np.uint8)))
    assert len(inst) == 576
    recs = {r: torch.from_numpy(np.ascontiguousarray(traces[r].rec).view(np.uint8).reshape(steps, -1)).cuda()
            for r in range(replicas)}
    ridx = [r for r in range(replicas) for _ in budgets]
    nonempty = 0
    for s in range(steps):
        for it, r in zip(inst, ridx):
            it["pl"].set_inputs_ptr(recs[r][s].data_ptr())
        step_batch([it["pl"] for it in inst], int(traces[0].now[s]))
        torch.cuda.synchronize()
        for i, it in enumerate(inst):
            w = it["w"]
            hdr = it["pl"].sync()
            d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
            p = oracle.plan(w.rec[s], d, it["res"], w.theta, it["budget"])
            assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"], (s, i)
            assert hdr["kept_bytes"] == p["kept_bytes"] and hdr["bytes_h2d"] == p["bytes_h2d"], (s, i)
            assert hdr["n_eligible"] == p["n_eligible"], (s, i)
            assert (hdr["status"] & oracle.ST_INSUFFICIENT) == (p["status"] & oracle.ST_INSUFFICIENT), (s, i)
            pf, ev = it["pl"].lists(hdr)
            assert np.array_equal(pf, p["prefetch"]) and np.array_equal(ev, p["evict"]), (s, i)
            assert np.array_equal(it["pl"].resident(), p["resident"]), (s, i)
            nonempty += int(len(pf) > 0) + int(len(ev) > 0)
            it["res"] = p["resident"]
    assert nonempty > 576  # the lists are exercised, not empty
    for it in inst:
        it["pl"].close()


def test_back_to_back_transfers_keep_writebacks_ordered():
    """No host sync between steps: step t's loads into pages released by step t-1 must not
    overtake step t-1's write-backs of those pages (copy_stream2 ordering)."""
    import torch
    from gpu_harness import make_planner
    P = tg.PAGE_BYTES
    w = tg.config_c2(seed=7, steps=12, n=2000, lora=2 * P, kv=P)
    n = w.n
    rng = np.random.default_rng(3)
    res0 = (rng.random(n) < 0.2).astype(np.uint8)
    # keep the initially resident set within the budget (the oracle's walk decides from there)
    fp = w.footprint.astype(np.int64)
    order = np.nonzero(res0)[0]
    keep = order[np.cumsum(fp[order]) <= w.budget]
    res0[:] = 0
    res0[keep] = 1
    pl = make_planner(w, transfer=True, resident_init=res0)
    b = w.blocks
    pages = max((w.budget + w.page_bytes - 1) // w.page_bytes, 1)
    om = oracle.OracleMem(b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, P, pages, resident_init=res0)
    torch.cuda.synchronize()
    # stamp every device page with a tag unlike any host pattern word
    n_dev = pl.dev_arena.numel() // P
    tags = np.stack([np.full(n_dev, 0xA11CE000, np.uint32) + np.arange(n_dev, dtype=np.uint32),
                     np.arange(n_dev, dtype=np.uint32), np.full(n_dev, 0x0BADF00D, np.uint32),
                     np.full(n_dev, 0x5EED5EED, np.uint32)], axis=1)
    dev_words = pl.dev_arena.view(torch.int32).view(n_dev, P // 4)
    dev_words[:, :4].copy_(torch.from_numpy(tags.view(np.int32)))
    torch.cuda.synchronize()
    # model of the first 16 bytes of every device page / written-back host range
    dev_tag = {pg: tags[pg].copy() for pg in range(n_dev)}
    host_tag = {}
    res = res0.copy()
    recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(w.steps, -1)).cuda()
    torch.cuda.synchronize()
    for s in range(w.steps):  # back to back: no host sync, no readback
        pl.set_inputs_ptr(recs[s].data_ptr())
        pl.step(int(w.now[s]))
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        mo = om.apply(w.rec[s], p["prefetch"], p["evict"])
        for ho, pg in zip(mo["d2h_host"], mo["d2h_page"]):  # write-backs first (R13), then loads
            host_tag[int(ho)] = dev_tag[int(pg)].copy()
        for ho, pg in zip(mo["h2d_host"], mo["h2d_page"]):
            ho = int(ho)
            dev_tag[int(pg)] = host_tag.get(ho, tg.host_pattern(16, seed=0, word_offset=ho // 4))
        res = p["resident"]
    hdr = pl.sync()
    assert hdr["status"] & oracle.ST_NO_PAGES == 0
    assert len(host_tag) > 20, len(host_tag)
    host = pl.host_arena
    for ho, tag in host_tag.items():
        got = host[ho:ho + 16].numpy().view(np.uint32)
        assert np.array_equal(got, tag), (ho, got, tag)
    # and the resident device pages hold what the model says
    pt = om.page_table()
    for q in np.nonzero(pt != 0xFFFFFFFF)[0][:256]:
        pg = int(pt[q])
        got = pl.dev_arena[pg * P:pg * P + 16].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, dev_tag[pg]), (q, pg, got, dev_tag[pg])
    pl.close()
