"""Debug: step the streaming kernel on C4 at 2.5M agents against the oracle; print the header
status of each step and the first differences."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import tracegen as tg  # noqa: E402
from gpu_harness import make_planner  # noqa: E402
from paper_2601_21473_b200 import _lib as L  # noqa: E402

n = int(os.environ.get("N", "2500000"))
w = tg.config_c4(seed=3, steps=6, n=n)
pl = make_planner(w, False, None, keep_dist=False)
print("big", pl.big)
res = np.zeros(n, np.uint8)
for s in range(w.steps):
    pl.set_records(w.rec[s])
    pl.step(int(w.now[s]))
    h = L.PlanHost()
    pl.lib.scalesim_sync(pl.ctx, C.byref(h))
    hd = h.as_dict()
    d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
    p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
    print("step", s, "status", hd["status"], "npf", hd["n_prefetch"], "vs", len(p["prefetch"]), "nev", hd["n_evict"], "vs",
          len(p["evict"]), "cut", hd["cut_bits"], p["cut_bits"])
    if hd["status"] == 0:
        pf, ev = pl.lists(hd)
        print("   pf equal", np.array_equal(pf, p["prefetch"]), "ev equal", np.array_equal(ev, p["evict"]))
        if not np.array_equal(ev, p["evict"]):
            k = np.nonzero(ev[:len(p["evict"])] != p["evict"][:len(ev)])[0][:5]
            print("   ev diff at", k, ev[k], p["evict"][k])
    res = pl.resident() if hd["status"] == 0 else p["resident"]
pl.close()
