"""Test-side driver: runs the CUDA planner (through the C ABI binding) and the CPU oracle
on the same seeded workload, step by step, and compares them element by element.

Parity bar: distances bit-identical (the north star's 1e-6 absolute bound is
asserted as well); resident sets, prefetch/evict lists, byte totals, boundary (D*, rem),
status bits, page assignment and copy descriptors bit-exact; arena contents equal to the
host bytes they were loaded from.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import tracegen as tg

ST_MASK = oracle.ST_INSUFFICIENT | oracle.ST_BAD_RECORD | oracle.ST_BAD_KIN | oracle.ST_NO_PAGES


def fill_pattern(host, chunk=1 << 28):
    """Per-offset pattern into a pinned host tensor, chunk by chunk (bounded host memory)."""
    hb = host.numel()
    words = host[: hb // 4 * 4].view(torch.int32)
    for o in range(0, hb // 4, chunk // 4):
        n = min(chunk // 4, hb // 4 - o)
        pat = tg.host_pattern(4 * n, seed=0, word_offset=o)
        words[o:o + n].copy_(torch.from_numpy(pat.view(np.int32)))


def make_planner(w: tg.Workload, transfer: bool, resident_init=None, host_pattern=True, dev_pages=None,
                 multi_kernel=False, explicit=False, keep_dist=True, stream=None, exclusive=False):
    from paper_2601_21473_b200.planner import Planner
    b = w.blocks
    host = None
    if transfer:
        hb = int(b.host_bytes)
        host = torch.empty(hb, dtype=torch.uint8, pin_memory=True)
        if host_pattern:
            fill_pattern(host)
    pages = dev_pages if dev_pages is not None else (w.budget + w.page_bytes - 1) // w.page_bytes
    return Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta,
                   hop_scale=w.hop_scale, n_kin=w.n_kin, page_bytes=w.page_bytes, transfer=transfer,
                   host_arena=host, dev_bytes=max(pages, 1) * w.page_bytes, resident_init=resident_init,
                   multi_kernel=multi_kernel, explicit_dist=explicit, keep_dist=keep_dist, stream=stream,
                   exclusive=exclusive)


def run_parity(w: tg.Workload, steps=None, transfer=True, resident_init=None, content_pages=64,
               check_dist=True, stamp_writes=True, seed=0, multi_kernel=False, expect_fused=None, explicit=False,
               keep_dist=True, exclusive=False):
    """Step the GPU planner and the oracle through the workload; assert parity every step.
    keep_dist=False is the bench's configuration (the fused kernel's fast P1 variant, no
    distance copy): distances are then compared through the plan (D*, lists, bytes) only.
    Returns per-step summaries."""
    pl = make_planner(w, transfer, resident_init, multi_kernel=multi_kernel, explicit=explicit, keep_dist=keep_dist,
                      exclusive=exclusive)
    check_dist = check_dist and keep_dist
    if expect_fused is None:
        expect_fused = not multi_kernel
    assert pl.fused == expect_fused
    res = np.zeros(w.n, np.uint8) if resident_init is None else np.asarray(resident_init, np.uint8).copy()
    om = None
    if transfer:
        b = w.blocks
        pages = max((w.budget + w.page_bytes - 1) // w.page_bytes, 1)
        om = oracle.OracleMem(b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.page_bytes, pages,
                              resident_init=res)
        page_first = np.concatenate([[0], np.cumsum(b.blk_size.astype(np.int64) // w.page_bytes)])
    rng = np.random.default_rng(seed)
    out = []
    steps = range(w.steps) if steps is None else steps
    P = w.page_bytes
    for s in steps:
        rec = w.rec[s]
        kin = w.kin[s] if w.kin is not None else None
        stamped = {}
        if transfer and stamp_writes:
            # simulate KV / history writes of dirty resident agents: stamp device pages
            pt = om.page_table()
            dirty = np.nonzero(((rec[:, 2] >> 4) & 1).astype(bool) & res.astype(bool))[0]
            for a in rng.permutation(dirty)[:8]:
                for blk in range(int(w.blocks.blk_ptr[a]), int(w.blocks.blk_ptr[a + 1])):
                    if w.blocks.blk_kind[blk] == tg.KIND_LORA:
                        continue
                    for q in range(int(page_first[blk]), int(page_first[blk + 1])):
                        pg = int(pt[q])
                        mark = np.array([0x5EED0000 + s, pg, a, q], np.uint32)
                        pl.dev_arena[pg * P: pg * P + 16].copy_(torch.from_numpy(mark.view(np.uint8)))
                        stamped[pg] = mark
            torch.cuda.synchronize()
        pl.set_records(rec, kin)
        pl.step(int(w.now[s]))
        hdr = pl.sync()
        # --- score parity
        if explicit:  # records carry their distances (R19)
            d_or, st_or = oracle.explicit_dist(rec)
        else:
            d_or, st_or = oracle.score(rec, kin, int(w.now[s]), w.hop_scale)
        if check_dist:
            d_gpu = pl.distances()
            bad = np.nonzero(d_gpu.view(np.uint32) != d_or.view(np.uint32))[0]
            assert len(bad) == 0, (s, bad[:10], d_gpu[bad[:10]], d_or[bad[:10]])
            fin = np.isfinite(d_or)
            assert np.all(np.abs(d_gpu[fin] - d_or[fin]) <= 1e-6)
        # --- plan parity
        p = oracle.plan(rec, d_or, res, w.theta, w.budget)
        status_or = (p["status"] | st_or) & ST_MASK
        assert (hdr["status"] & ~oracle.ST_NO_PAGES) == status_or, (s, hdr["status"], status_or)
        assert hdr["n_prefetch"] == len(p["prefetch"]) and hdr["n_evict"] == len(p["evict"]), (s, hdr, len(p["prefetch"]), len(p["evict"]))
        assert hdr["cut_bits"] == p["cut_bits"], (s, hex(hdr["cut_bits"]), hex(p["cut_bits"]))
        assert hdr["cut_rem"] == p["cut_rem"], (s, hdr["cut_rem"], p["cut_rem"])
        assert hdr["bytes_h2d"] == p["bytes_h2d"]
        assert hdr["kept_bytes"] == p["kept_bytes"], (s, hdr["kept_bytes"], p["kept_bytes"])
        assert hdr["n_eligible"] == p["n_eligible"]
        pf, ev = pl.lists(hdr)
        assert np.array_equal(pf, p["prefetch"]), (s, pf[:10], p["prefetch"][:10])
        assert np.array_equal(ev, p["evict"]), (s, ev[:10], p["evict"][:10])
        assert np.array_equal(pl.resident(), p["resident"])
        # --- write-back bytes (R13) are accounted in every mode
        dirty = ((rec[:, 2] >> 4) & 1).astype(bool)
        wb = 0
        b = w.blocks
        for a in p["evict"]:
            if dirty[a]:
                k = b.blk_kind[int(b.blk_ptr[a]):int(b.blk_ptr[a + 1])]
                z = b.blk_size[int(b.blk_ptr[a]):int(b.blk_ptr[a + 1])]
                wb += int(z[k != tg.KIND_LORA].astype(np.int64).sum())
        assert hdr["bytes_d2h"] == wb
        if transfer:
            mo = om.apply(rec, p["prefetch"], p["evict"])
            assert mo["bytes_d2h"] == hdr["bytes_d2h"]
            assert hdr["n_d2h"] == len(mo["d2h_page"]) and hdr["n_h2d"] == len(mo["h2d_page"])
            d2h, h2d = pl.descriptors(hdr)
            assert np.array_equal(d2h[:, 0], mo["d2h_host"]) and np.array_equal(d2h[:, 1], mo["d2h_page"])
            assert np.array_equal(h2d[:, 0], mo["h2d_host"]) and np.array_equal(h2d[:, 1], mo["h2d_page"])
            assert np.array_equal(pl.page_table(), om.page_table())
            head, tail, _ = om.pool()
            assert hdr["pool_head"] == head and hdr["pool_tail"] == tail
            # content: loaded pages equal their host bytes; written-back pages carry the stamp
            host = pl.host_arena
            idx = rng.permutation(len(h2d))[:content_pages]
            for k in idx:
                ho, pg = int(h2d[k, 0]), int(h2d[k, 1])
                dev = pl.dev_arena[pg * P:(pg + 1) * P].cpu()
                assert torch.equal(dev, host[ho:ho + P]), (s, k, ho, pg)
            for k in range(len(d2h)):
                ho, pg = int(d2h[k, 0]), int(d2h[k, 1])
                if pg in stamped:
                    got = host[ho:ho + 16].numpy().view(np.uint32)
                    assert np.array_equal(got, stamped[pg]), (s, k, got, stamped[pg])
        res = p["resident"]
        out.append(dict(step=s, n_prefetch=len(p["prefetch"]), n_evict=len(p["evict"]),
                        bytes_h2d=p["bytes_h2d"], status=hdr["status"]))
    if pl.fused and out:  # fused launches that took the fast / the two-barrier list placement
        out[-1]["paths"] = pl.list_paths()
    pl.close()
    return out
