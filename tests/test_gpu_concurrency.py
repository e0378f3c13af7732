"""Two fused contexts on two streams stepping concurrently: the fused
plan kernel's grid barrier needs all of its CTAs resident; the cooperative launch makes a
second context's kernel wait for SMs instead of spinning on absent CTAs.  Runs in a child
process under a timeout, so a deadlock fails the test instead of hanging the GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + '/tests')
import oracle, tracegen as tg
from gpu_harness import make_planner
ws = [tg.config_c4(seed=11, steps=8, n=300_000), tg.config_c4(seed=12, steps=8, n=250_000)]
pls = [make_planner(w, transfer=False, keep_dist=False, exclusive=EXCL) for w in ws]
assert pls[0].stream.cuda_stream != pls[1].stream.cuda_stream
assert all(pl.fused for pl in pls)
recs = [torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(w.steps, -1)).cuda() for w in ws]
torch.cuda.synchronize()
for s in range(8):  # interleaved, never synchronised: both streams hold plan kernels at once
    for pl, w, r in zip(pls, ws, recs):
        pl.set_inputs_ptr(r[s].data_ptr())
        pl.step(int(w.now[s]))
for pl, w in zip(pls, ws):
    hdr = pl.sync()
    res = np.zeros(w.n, np.uint8)
    for s in range(8):
        d, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
        res = p["resident"]
    pf, ev = pl.lists(hdr)
    assert np.array_equal(pf, p["prefetch"]) and np.array_equal(ev, p["evict"])
    assert np.array_equal(pl.resident(), p["resident"]) and hdr["cut_bits"] == p["cut_bits"]
    assert hdr["seq"] == 8, hdr["seq"]
print("CONCURRENT_OK")
"""


@pytest.mark.parametrize("exclusive", [False, True], ids=["cooperative", "exclusive-chained"])
def test_two_contexts_two_streams_concurrently(exclusive):
    """Default contexts launch cooperatively; SCALESIM_F_EXCLUSIVE contexts are ordered by the
    library's per-device event chain."""
    code = CHILD.replace("ROOT", repr(ROOT)).replace("EXCL", repr(exclusive))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "CONCURRENT_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
