"""Phase stamps of the streaming kernel (large contexts) on the replicated C4 population."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tracegen as tg  # noqa: E402
from paper_2601_21473_b200.planner import Planner  # noqa: E402

m = int(os.environ.get("M", "16"))
n = m * 1_000_000
w1 = tg.config_c4(seed=1, steps=12, n=1_000_000)
fp1 = np.ascontiguousarray(w1.rec[0][:, 1]).astype(np.uint32)
dev = torch.device("cuda", 0)
recs = [torch.from_numpy(np.ascontiguousarray(w1.rec[s]).view(np.uint8).reshape(-1, 16)).to(dev).repeat(m, 1).reshape(-1)
        for s in range(12)]
pl = Planner(n, np.arange(n + 1, dtype=np.uint64), np.tile(fp1, m), np.zeros(n, np.uint64),
             np.full(n, tg.KIND_KV, np.uint8), m * w1.budget, w1.theta, transfer=False, keep_dist=False, exclusive=True)
print("big", pl.big)
for s in range(12):
    pl.stamps(reset=True)
    pl.set_inputs_ptr(recs[s].data_ptr())
    pl.step(int(w1.now[s]))
    h = pl.sync()
    st = pl.stamps().astype(np.int64)
    if s >= 8:
        r = lambda q: round((int(st[q]) - int(st[0])) / 1e3, 1) if st[q] else None  # noqa: E731
        print(f"step {s}: us P1 {r(25)} pub {r(26)} B1 {r(4)} sel+own {r(41)} pos {r(17)} P34 {r(39)} end {r(1)} | "
              f"P34 parts (max over CTAs, us): a {st[22]/1e3:.1f} b {st[23]/1e3:.1f} c {st[24]/1e3:.1f} d {st[29]/1e3:.1f} "
              f"| npf {h['n_prefetch']} nev {h['n_evict']} | sort ns max (pf, ev) {st[50]} {st[51]} n max {st[52]} {st[53]}")
pl.close()
