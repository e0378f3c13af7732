"""Small parity runs for compute-sanitizer (memcheck / racecheck / synccheck): C1 variants,
a C2 mini with physical transfers, a tie-cut case, both plan paths, fused keep / no-keep."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import tracegen as tg  # noqa: E402
from gpu_harness import run_parity  # noqa: E402

for mk in (False, True):
    for variant in ("ind", "int", "diff"):
        w = tg.config_c1(seed=1, theta=(3.0, 3.0, 3.0), variant=variant)
        run_parity(w, multi_kernel=mk)
    w = tg.config_c2(seed=2, steps=4, n=1200, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    run_parity(w, multi_kernel=mk)
    run_parity(w, transfer=False, multi_kernel=mk, keep_dist=False)
# the streaming kernel of large contexts (a small tile forced: 150k agents on 4 CTAs would not
# exercise it; a 2.1M-agent C4 shard does) and a loopback world
w = tg.config_c4(seed=3, steps=2, n=2_100_000)
run_parity(w, transfer=False, keep_dist=False)
# the host entry points: staged whole records, incremental updates (synchronous and submitted,
# three in flight), the read-back kernel
import torch  # noqa: E402
from gpu_harness import make_planner  # noqa: E402
w = tg.config_c4(seed=4, steps=6, n=40_000)
pl = make_planner(w, transfer=False, keep_dist=False)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
pf = np.zeros(w.n, np.uint32)
ev = np.zeros(w.n, np.uint32)
r = [pin(w.rec[s]) for s in range(w.steps)]
pl.stage_host(r[0])
pl.stage_host(r[1])
pl.step_host(int(w.now[0]), r[0], None, pf, ev)
pl.step_host(int(w.now[1]), r[1], None, pf, ev)
upd = [None] + [(pin(np.nonzero(np.any(w.rec[s] != w.rec[s - 1], axis=1))[0].astype(np.uint32)), None)
                for s in range(1, w.steps)]
upd = [None] + [(u[0], pin(w.rec[s][u[0]])) for s, u in enumerate(upd) if u is not None]
pl.step_updates(int(w.now[2]), *upd[2], pf, ev)
for s in (3, 4, 5):
    pl.submit_updates(int(w.now[s]), *upd[s])
for s in (3, 4, 5):
    pl.collect(pf, ev)
pl.close()
print("SANITIZE_RUN_OK")
