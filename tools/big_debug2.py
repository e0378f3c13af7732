"""Debug: eligible counts of the streaming kernel, P1 side vs P34 side (DEBUG_WMASK build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import tracegen as tg  # noqa: E402
from gpu_harness import make_planner  # noqa: E402

n = int(os.environ.get("N", "2500000"))
w = tg.config_c4(seed=3, steps=3, n=n)
pl = make_planner(w, False, None, keep_dist=True)
res = np.zeros(n, np.uint8)
for s in range(w.steps):
    pl.stamps(reset=True)
    pl.set_records(w.rec[s])
    pl.step(int(w.now[s]))
    hd = pl.sync()
    st = pl.stamps().astype(np.int64)
    d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
    el = (res == 1) | (d == 0) | (d < w.theta[0])
    print("step", s, "hdr n_elig", hd["n_eligible"], "oracle", int(el.sum()), "P1 ballots", st[63], "P1 elig", st[61], "P34", st[62])
    res = pl.resident()
pl.close()
