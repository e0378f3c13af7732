"""Checks of the synthetic workload generator against SPEC's workload examples."""
import numpy as np

import tracegen as tg


def test_bfs_path_and_star():
    """path A-B-C, source A -> activation order A, B, C; star, source = centre ->
    all leaves at once."""
    adj = [[1], [0, 2], [1]]
    assert tg.bfs_hops(adj, [0]).tolist() == [0, 1, 2]
    star = [[1, 2, 3, 4, 5]] + [[0]] * 5
    assert tg.bfs_hops(star, [0]).tolist() == [0, 1, 1, 1, 1, 1]
    assert tg.bfs_hops([[1], [0], []], [0]).tolist() == [0, 1, tg.UNREACHABLE]


def test_diffusion_order_follows_hops():
    """activation order respects non-decreasing hop count (uniform delays), checked
    against an independent BFS (here: a dense-matrix power iteration)."""
    n = 50
    adj = tg.ba_graph(n, 2, seed=3)
    A = np.zeros((n, n), bool)
    for u, nb in enumerate(adj):
        A[u, nb] = True
    src = [0]
    hop = np.full(n, -1)
    frontier = np.zeros(n, bool)
    frontier[src] = True
    seen = frontier.copy()
    level = 0
    while frontier.any():
        hop[frontier] = level
        nxt = A[frontier].any(0) & ~seen
        seen |= nxt
        frontier = nxt
        level += 1
    assert np.array_equal(tg.bfs_hops(adj, src), np.where(hop < 0, tg.UNREACHABLE, hop))
    P, T, D = tg.gen_diffusion(n, 40, seed=1, adj=adj, sources=src, period=2)
    first = np.full(n, -1)
    for s in range(40):
        act = (P[s] == tg.PH_WAITING) & (first < 0)
        first[act] = s
    reached = first >= 0
    order = np.argsort(first[reached], kind="stable")
    assert np.all(np.diff(hop[reached][order]) >= 0)


def test_independent_active_rate():
    """target active rate reached statistically (here 5% and 20%)."""
    for rate in (0.05, 0.2):
        P, T, D = tg.gen_independent(5000, 60, seed=2, active=rate)
        frac = np.mean(P[10:] != tg.PH_ACTING)
        assert abs(frac - rate) < 0.35 * rate


def test_independent_exactness():
    """with known durations the remaining action duration equals the true time until
    the agent's next request (checked on the generated trace)."""
    P, T, D = tg.gen_independent(300, 80, seed=4, fixed_dur=(2, 9), g_choices=(1, 2))
    for s in range(60):
        acting = P[s] == tg.PH_ACTING
        for a in np.nonzero(acting)[0][:50]:
            nxt = next(u for u in range(s, 80) if P[u, a] == tg.PH_WAITING)
            assert T[s, a] == nxt


def test_records_and_blocks_layout():
    w = tg.config_c3(seed=1, steps=2, n=300)
    assert w.rec.dtype == np.uint32 and w.rec.shape == (2, 300, 4)
    fp = w.blocks.footprint
    assert np.array_equal(fp, w.rec[0, :, 1].astype(np.uint64))
    assert np.all(w.blocks.blk_size % tg.PAGE_BYTES == 0)
    cls = (w.rec[0, :, 2] >> 2) & 3
    assert set(np.unique(cls).tolist()) == {0, 1, 2}
    ki = w.rec[0, cls == 1, 3]
    assert np.array_equal(ki, np.arange(len(ki)))


def test_noise_knob_estimates_only():
    """the noise knob perturbs only the recorded action ends (the estimates); phases
    (the true lifecycle) are unchanged, noise 0 reproduces the exact trace, and the estimate
    error of an action is lognormal with the knob's sigma (up to rounding)."""
    P0, T0, D0 = tg.gen_independent(20000, 30, seed=3)
    Pz, Tz, Dz = tg.gen_independent(20000, 30, seed=3, noise=0.0)
    assert np.array_equal(P0, Pz) and np.array_equal(T0, Tz) and np.array_equal(D0, Dz)
    P1, T1, D1 = tg.gen_independent(20000, 30, seed=3, noise=0.5)
    assert np.array_equal(P0, P1) and np.array_equal(D0, D1)
    acting = P0 == tg.PH_ACTING
    assert np.array_equal(T0[~acting], T1[~acting])
    assert (T0[acting] != T1[acting]).mean() > 0.3
    # per action (first step an agent is ACTING after an LLM phase): log(est / true) duration
    s = 5
    start = acting[s] & ~acting[s - 1]
    true = (T0[s, start] - s).astype(float)
    est = (T1[s, start] - s).astype(float)
    big = true >= 20  # (rounding negligible)
    r = np.log(est[big] / true[big])
    assert abs(r.mean()) < 0.05 and abs(r.std() - 0.5) < 0.05, (r.mean(), r.std(), big.sum())
