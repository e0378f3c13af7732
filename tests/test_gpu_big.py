"""Large contexts: more agents per SM than the shared-memory tile holds
(> 12288 per CTA) plan with the streaming single-kernel variant (fused_big.cu, scalesim_fused
== 2).  Parity with the oracle at 2.5M and 16M agents (C4 shape: the population of
independent agents of config_c4 with its 1M-agent statistics), a tie group cut across CTAs
at 3M agents, the distance view, and the documented limit (D* >= 2048 ticks: SCALESIM_ST_LIMIT)."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import rec_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


@pytest.mark.parametrize("n,steps,keep", [pytest.param(2_500_000, 8, False, id="2.5M"),
                                          pytest.param(2_500_000, 3, True, id="2.5M-keepdist"),
                                          pytest.param(16_000_000, 3, False, id="16M")])
def test_big_c4_parity(n, steps, keep):
    from gpu_harness import run_parity
    w = tg.config_c4(seed=3, steps=steps, n=n)
    out = run_parity(w, transfer=False, keep_dist=keep)
    assert out[-1]["n_prefetch"] > 0


def test_big_mode_is_used_and_ties_cut_across_ctas():
    from gpu_harness import make_planner, run_parity
    n = 3_000_000
    rng = np.random.default_rng(4)
    fp = (rng.choice([1, 2, 3], n) * tg.PAGE_BYTES).astype(np.uint32)
    d = np.where(rng.random(n) < 0.7, 5, rng.integers(0, 40, n))
    rec = tg.pack_records(d, fp, np.zeros(n, np.int64), np.zeros(n, np.int64), (rng.random(n) < 0.5).astype(np.int64),
                          np.zeros(n, np.int64))[None]
    from tracegen import traces as tgt
    blocks = tgt._blocks_vectorized(n, 0, tg.PAGE_BYTES, (fp // tg.PAGE_BYTES).astype(np.int64), 0, None)
    below = int(fp[d < 5].astype(np.int64).sum())
    tie = np.nonzero(d == 5)[0]
    cs = np.cumsum(fp[tie].astype(np.int64))
    for j in (len(tie) // 3, len(tie) // 2 + 7):
        w = tg.Workload("bigties", n, np.array([0]), rec, None, blocks, below + int(cs[j]), np.full(3, 50.0, np.float32))
        pl = make_planner(w, transfer=False, keep_dist=False)
        assert pl.big
        pl.close()
        run_parity(w, transfer=False, keep_dist=False, resident_init=(rng.random(n) < 0.4).astype(np.uint8))


def test_big_limit_status():
    """Distances >= 2048 ticks at the boundary are outside the streaming kernel's scope: the
    plan reports SCALESIM_ST_LIMIT (sync returns E_INVARIANT) instead of a wrong plan."""
    from gpu_harness import make_planner
    from paper_2601_21473_b200 import _lib as L
    n = 2_000_000
    rng = np.random.default_rng(5)
    agents_d = rng.integers(3000, 100000, n)
    rec = tg.pack_records(agents_d, np.full(n, tg.PAGE_BYTES), np.zeros(n, np.int64), np.zeros(n, np.int64),
                          np.zeros(n, np.int64), np.zeros(n, np.int64))[None]
    from tracegen import traces as tgt
    blocks = tgt._blocks_vectorized(n, 0, tg.PAGE_BYTES, np.ones(n, np.int64), 0, None)
    w = tg.Workload("far", n, np.array([0]), rec, None, blocks, n * tg.PAGE_BYTES // 3, np.full(3, np.inf, np.float32))
    pl = make_planner(w, transfer=False, keep_dist=False)
    assert pl.big
    pl.set_records(rec[0])
    pl.step(0)
    with pytest.raises(L.ScaleSimError) as e:
        pl.sync()
    assert e.value.status == L.E_INVARIANT
    import ctypes as C
    h = L.PlanHost()
    pl.lib.scalesim_sync(pl.ctx, C.byref(h))
    assert h.as_dict()["status"] & 32  # SCALESIM_ST_LIMIT
    pl.close()
