"""C3 with physical transfers, steps back to back: per step, the planner stream's plan interval
and the copy stream's transfer interval (device events), cooperative vs exclusive launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tracegen as tg  # noqa: E402
from paper_2601_21473_b200.planner import Planner  # noqa: E402

warm, steps = 3, 6
T = warm + steps
w = tg.config_c3(seed=1, steps=T, host_bytes=8 << 30)
b = w.blocks
dev = torch.device("cuda", 0)
recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(T, -1)).to(dev)
kins = torch.from_numpy(np.ascontiguousarray(w.kin).view(np.uint8).reshape(T, -1)).to(dev)
host = torch.empty(int(b.host_bytes), dtype=torch.uint8, pin_memory=True)
for excl in (False, True):
    pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, hop_scale=w.hop_scale,
                 n_kin=w.n_kin, page_bytes=w.page_bytes, transfer=True, host_arena=host, keep_dist=False,
                 exclusive=excl)
    for s in range(warm):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        pl.step(int(w.now[s]))
    pl.sync()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    e0 = ev()
    pa, ps, pb, xa, xe = ([ev() for _ in range(steps)] for _ in range(5))
    e0.record(pl.stream)
    for k, s in enumerate(range(warm, T)):
        pl.set_inputs_ptr(recs[s].data_ptr(), kins[s].data_ptr())
        pa[k].record(pl.stream)
        pl.score(int(w.now[s]))
        ps[k].record(pl.stream)
        pl.plan()
        pb[k].record(pl.stream)
        xa[k].record(pl.copy_stream)
        pl.transfer()
        xe[k].record(pl.copy_stream)
    pl.join()
    torch.cuda.synchronize()
    print("exclusive" if excl else "cooperative", "fused", pl.fused)
    for k in range(steps):
        t = lambda e: round(e0.elapsed_time(e), 3)  # noqa: E731
        print(f"  step {k}: plan [{t(pa[k])}, score {t(ps[k])}, {t(pb[k])}] transfer [{t(xa[k])}, {t(xe[k])}]")
    pl.close()
