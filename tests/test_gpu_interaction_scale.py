"""NEXT #4 at scale: the exact spatially pruned interaction scoring (a1', Eq. 2) on 10^6
interaction agents (Generative-Agents-style movement in a proportionally larger arena).  The
oracle's O(n^2) scan is out of reach at this size, so 2,000 sampled agents are scored by the
oracle against every other participant (oracle.score_sampled) and compared bit for bit with the
GPU's distances of the same step."""
import numpy as np
import pytest

import oracle
import tracegen as tg
from tracegen import traces as tgt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


def interaction_workload(n, steps, seed):
    arena = 2000.0 * np.sqrt(n / 33_333.0)
    P, T, D, K = tg.gen_interaction(n, steps, seed, active=0.05, arena=arena)
    blocks = tgt._blocks_vectorized(n, tg.PAGE_BYTES, tg.PAGE_BYTES, np.ones(n, np.int64), 0, None)
    fp = blocks.footprint
    return tgt._assemble("int1m", P, T, D, np.full(n, tg.CL_INT), fp, blocks, int(fp.sum()) // 4, (4.0, 4.0, 4.0),
                        kin=K, kin_idx=np.arange(n, dtype=np.uint32))


def test_grid_interaction_1m_agents_sampled_parity():
    import torch
    from gpu_harness import make_planner
    n = 1_000_000
    w = interaction_workload(n, 2, seed=31)
    pl = make_planner(w, transfer=False, keep_dist=True)
    rng = np.random.default_rng(2)
    for s in range(w.steps):
        pl.set_records(w.rec[s], w.kin[s])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(pl.stream)
        pl.score(int(w.now[s]))
        e1.record(pl.stream)
        pl.plan()
        pl.sync()
        d_gpu = pl.distances()
        acting = np.nonzero((w.rec[s][:, 2] & 3) == tg.PH_ACTING)[0]
        idx = np.sort(np.concatenate([rng.choice(acting, 1500, replace=False), rng.choice(n, 500, replace=False)]))
        d_or, _ = oracle.score_sampled(w.rec[s], w.kin[s], int(w.now[s]), idx)
        bad = np.nonzero(d_gpu[idx].view(np.uint32) != d_or.view(np.uint32))[0]
        assert len(bad) == 0, (s, idx[bad[:5]], d_gpu[idx[bad[:5]]], d_or[bad[:5]])
        # the sample exercises the pair term: some sampled distances come from Eq. 2, not D_action
        d_act = np.maximum(0, w.rec[s][idx, 0].astype(np.int64) - int(w.now[s])).astype(np.float32)
        acting_s = (w.rec[s][idx, 2] & 3) == tg.PH_ACTING
        assert ((d_or < d_act) & acting_s).sum() > 10
        print(f"step {s}: a1' (interaction scoring, 1e6 agents, {len(acting)} acting) {e0.elapsed_time(e1):.3f} ms")
    pl.close()
