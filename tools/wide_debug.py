"""Debug: the `wide` workload (distances 16..19, one list bucket) in a batch of 80 single-CTA
instances vs the oracle, per step: cut bits, kept bytes, lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, tracegen as tg
from helpers import rec_of
from paper_2601_21473_b200.planner import Planner, step_batch
n, steps = 1500, 4
rng = np.random.default_rng(5)
fpw = rng.choice([1, 2], n) * tg.PAGE_BYTES
recw = np.stack([rec_of([dict(d=int(rng.integers(16, 20)), fp=int(fpw[a]), dirty=int(rng.integers(0, 2)))
                         for a in range(n)]) for _ in range(steps)])
blw = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fpw])
theta = np.full(3, 50.0, np.float32)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 80
stream = torch.cuda.Stream()
pcts = [10 * (1 + i % 9) for i in range(K)]
pls = [Planner(n, blw.blk_ptr, blw.blk_size, blw.blk_host_off, blw.blk_kind,
               int(blw.blk_size.astype(np.int64).sum()) * pcts[i] // 100, theta, transfer=False, stream=stream)
       for i in range(K)]
res = [np.zeros(n, np.uint8) for _ in range(K)]
for s in range(steps):
    for pl in pls:
        pl.set_records(recw[s])
    if K == 1:
        pls[0].step(0)
    else:
        step_batch(pls, 0)
    d, _ = oracle.score(recw[s], None, 0)
    bad = []
    for i, pl in enumerate(pls):
        h = pl.sync()
        p = oracle.plan(recw[s], d, res[i], theta, pl_budget := int(blw.blk_size.astype(np.int64).sum()) * pcts[i] // 100)
        pf, ev = pl.lists(h)
        ok = (h["cut_bits"] == p["cut_bits"], h["kept_bytes"] == p["kept_bytes"], np.array_equal(pf, p["prefetch"]),
              np.array_equal(ev, p["evict"]), np.array_equal(pl.resident(), p["resident"]))
        if not all(ok):
            bad.append((i, pcts[i], ok, h["cut_bits"], p["cut_bits"], h["kept_bytes"], p["kept_bytes"], len(pf), len(p["prefetch"])))
        res[i] = p["resident"]
    print("step", s, "bad", len(bad), bad[:4])
