"""The N>1 decomposition of the cut, exercised with world_size 2 over gloo on
CPU: agents shard by contiguous id; every rank builds byte-weighted radix histograms of its
eligible distance bits (digits 11/10/10), the histograms are all-gathered and summed
(exact u64), which fixes the boundary distance D* and the remaining budget; then one u64
per rank (its bytes at d == D*) is all-gathered and its exclusive prefix over ranks is the
id-order prefix of the tie group.  The union of the ranks' kept sets must equal the
oracle's global plan bit for bit.

The decomposition is written out here in numpy (test code); the CUDA path implements the
same exchange with NCCL on the device.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tracegen as tg

DIGITS = [(20, 11), (10, 10), (0, 10)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sharded_cut(dbits_elig, fp, budget, allgather):
    """dbits_elig: local u32 f32-bit keys (0xFFFFFFFF for non-eligible) in id order."""
    elig = dbits_elig != 0xFFFFFFFF
    prefix, plen, below = 0, 0, 0  # bits fixed so far, their count, bytes strictly below
    for shift, width in DIGITS:
        sel = elig & ((dbits_elig >> (shift + width)) == (prefix >> (shift + width))) if plen else elig
        digit = (dbits_elig[sel] >> shift) & ((1 << width) - 1)
        h = np.zeros(1 << width, np.uint64)
        np.add.at(h, digit, fp[sel].astype(np.uint64))
        hs = sum(allgather(h))  # exact u64 sum over ranks
        cum = np.cumsum(hs)
        over = np.nonzero(below + cum > budget)[0]
        if len(over) == 0:
            return 0xFFFFFFFF, budget - (below + int(cum[-1])), None
        b = int(over[0])
        below += int(cum[b - 1]) if b > 0 else 0
        prefix |= b << shift
        plen += width
    dstar = prefix
    rem = budget - below
    tie = elig & (dbits_elig == dstar)
    mine = np.uint64(fp[tie].astype(np.uint64).sum())
    per_rank = allgather(np.array([mine], np.uint64))
    return dstar, rem, per_rank


def worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allgather(arr):
        t = torch.from_numpy(arr.astype(np.int64))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [o.numpy().astype(np.uint64) for o in out]

    w = tg.config_c2(seed=seed, steps=12, n=1001)
    n = w.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    res = np.zeros(n, np.uint8)
    ok = True
    for s in range(w.steps):
        d, _ = oracle.score(w.rec[s], None, w.now[s])
        glob = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        fp = w.rec[s, :, 1].astype(np.uint64)
        el = (res != 0) | (d == 0) | (d < w.theta[0])
        bits = np.where(el, d.view(np.uint32), np.uint32(0xFFFFFFFF)).astype(np.uint64)
        dstar, rem, per_rank = sharded_cut(bits[lo:hi], fp[lo:hi], w.budget, allgather)
        kept = np.zeros(hi - lo, bool)
        loc_el = bits[lo:hi] != 0xFFFFFFFF
        if per_rank is None:
            kept = loc_el
        else:
            excl = int(sum(int(x[0]) for x in per_rank[:rank]))
            tie = loc_el & (bits[lo:hi] == dstar)
            incl = excl + np.cumsum(np.where(tie, fp[lo:hi], 0).astype(np.uint64))
            kept = loc_el & ((bits[lo:hi] < dstar) | (tie & (incl <= rem)))
        ok &= bool(np.array_equal(kept, glob["resident"][lo:hi].astype(bool)))
        ok &= (dstar == glob["cut_bits"]) and (rem == glob["cut_rem"])
        res = glob["resident"]
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 2])
def test_sharded_cut_gloo_world2(seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
