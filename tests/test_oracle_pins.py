"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it follows.  The oracle is never compared with itself: the
expected values come from the paper's worked examples (tests/golden/, cited), closed forms
in exact rational arithmetic, brute-force enumeration, an exhaustive offline optimum,
and textbook special cases (Belady's MIN).
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tracegen as tg
from helpers import rec_of, round_f32

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = np.float32(np.inf)


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def no_theta():
    return np.array([np.inf, np.inf, np.inf], np.float32)


# ----------------------------------------------------------------------------------------
# Score: Eq. 1, Eq. 2, phase rules


def test_eq2_worked_example():
    """S:173 [PAPER: Eq. (1)-(2)]: D_action=10, gap 12, closing speed 3 -> D = 4."""
    g = gold("eq2_example.json")
    now = 100
    agents = [dict(cls=tg.CL_INT, d=g["d_action"], kin=0), dict(cls=tg.CL_INT, d=1000, kin=1)]
    # agent 0 at rest at the origin, agent 1 at distance 12 moving toward it at speed 3
    kin = np.array([[0, 0, 0, 0], [g["gap"], 0, -g["closing_speed"], 0]], np.float32)
    d, st = oracle.score(rec_of(agents, now), kin, now)
    assert st == 0
    assert d[0] == np.float32(g["expected_d"])
    assert d[1] == np.float32(g["expected_d_interaction"])  # min(1000, 4)
    # the same encounter with both agents moving (closing speed still 3) and rotated
    kin2 = np.array([[5, -7, 0.0, 1.5], [5, 5, 0.0, -1.5]], np.float32)
    d2, _ = oracle.score(rec_of(agents, now), kin2, now)
    assert d2[0] == np.float32(4.0) and d2[1] == np.float32(4.0)


def test_eq2_not_approaching_is_infinite():
    """pairs with non-positive closing speed contribute +infinity -> D = D_action."""
    now = 0
    agents = [dict(cls=tg.CL_INT, d=7, kin=0), dict(cls=tg.CL_INT, d=9, kin=1), dict(cls=tg.CL_INT, d=3, kin=2)]
    kin = np.array([[0, 0, -1, 0], [10, 0, 1, 0], [0, 50, 0, 3]], np.float32)  # every pair diverging
    d, _ = oracle.score(rec_of(agents, now), kin, now)
    dint, _ = oracle.interaction(rec_of(agents, now), kin)
    assert np.all(np.isinf(dint))
    assert list(d) == [7.0, 9.0, 3.0]


def test_eq2_exact_rational_closed_form():
    """Eq. 2 on integer kinematics: every product and sum is exact in f32, so
    the distance must equal the correctly rounded rational min_j |r|^2/(-r.w) (the
    min over other ACTING agents, approaching pairs only)."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(2, 9))
        kin = np.concatenate([rng.integers(-60, 61, (n, 2)), rng.integers(-4, 5, (n, 2))], 1).astype(np.float32)
        agents = [dict(cls=tg.CL_INT, d=10 ** 6, kin=i) for i in range(n)]
        dint, st = oracle.interaction(rec_of(agents), kin)
        assert st == 0
        for i in range(n):
            best = None
            for j in range(n):
                if j == i:
                    continue
                r = [Fraction(int(kin[j, c] - kin[i, c])) for c in (0, 1)]
                w = [Fraction(int(kin[j, c + 2] - kin[i, c + 2])) for c in (0, 1)]
                rw = r[0] * w[0] + r[1] * w[1]
                if rw < 0:
                    t = (r[0] ** 2 + r[1] ** 2) / (-rw)
                    best = t if best is None else min(best, t)
            expect = INF if best is None else round_f32(best)
            assert dint[i] == expect, (trial, i, dint[i], expect)


def test_eq2_is_gap_over_closing_speed():
    """Eq. 2 reading R6: Physical Distance / Velocity with velocity = closing speed
    -d|r|/dt.  Check against a float64 finite difference of the gap |p_j - p_i|."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        kin = rng.uniform(-50, 50, (2, 4)).astype(np.float32)
        kin[:, 2:] = rng.uniform(-3, 3, (2, 2)).astype(np.float32)
        agents = [dict(cls=tg.CL_INT, d=10 ** 7, kin=0), dict(cls=tg.CL_INT, d=10 ** 7, kin=1)]
        dint, _ = oracle.interaction(rec_of(agents), kin)
        k = kin.astype(np.float64)
        gap = lambda t: np.hypot(k[1, 0] - k[0, 0] + t * (k[1, 2] - k[0, 2]), k[1, 1] - k[0, 1] + t * (k[1, 3] - k[0, 3]))
        h = 1e-6
        closing = -(gap(h) - gap(-h)) / (2 * h)
        if closing > 1e-3:
            assert dint[0] == pytest.approx(gap(0) / closing, rel=1e-4)
            assert dint[0] == dint[1]  # symmetric pair
        elif closing < -1e-3:
            assert np.isinf(dint[0])


def test_eq1_dominance_and_partners():
    """S:178 Eq. 1 dominance D <= D_action; partners are other ACTING INT agents only."""
    w = tg.config_c1(seed=3, variant="int")
    for s in range(w.steps):
        d, st = oracle.score(w.rec[s], w.kin[s], w.now[s])
        assert st == 0
        rec = w.rec[s]
        acting = (rec[:, 2] & 3) == tg.PH_ACTING
        d_action = np.maximum(0, rec[:, 0].astype(np.int64) - w.now[s]).astype(np.float32)
        assert np.all(d[acting] <= d_action[acting])
    # a non-acting INT agent never serves as partner; an IND agent never either
    agents = [dict(cls=tg.CL_INT, d=50, kin=0), dict(cls=tg.CL_INT, phase=tg.PH_GENERATING, kin=1),
              dict(cls=tg.CL_IND, d=50, kin=1)]
    kin = np.array([[0, 0, 0, 0], [2, 0, -1, 0]], np.float32)
    d, _ = oracle.score(rec_of(agents), kin, 0)
    assert list(d) == [50.0, 0.0, 50.0]


def test_phase_rules():
    """WAITING/GENERATING -> 0; IDLE -> +inf; independent -> remaining action
    duration (clamped at 0, R8); diffusion -> hop count x hop_scale, +inf if unreachable;
    S:174: diffusion agents at hops 1 and 2 -> distances 1 and 2."""
    now = 40
    agents = [
        dict(phase=tg.PH_WAITING, d=9), dict(phase=tg.PH_GENERATING, d=9), dict(phase=tg.PH_IDLE, d=9),
        dict(d=5), dict(d=0), dict(d=-3),
        dict(cls=tg.CL_DIFF, hop=1), dict(cls=tg.CL_DIFF, hop=2), dict(cls=tg.CL_DIFF, hop=tg.UNREACHABLE),
        dict(cls=tg.CL_DIFF, hop=3, phase=tg.PH_IDLE),
    ]
    d, st = oracle.score(rec_of(agents, now), None, now, hop_scale=1.0)
    assert st == 0
    assert list(d) == [0, 0, np.inf, 5, 0, 0, 1, 2, np.inf, np.inf]
    assert all(np.float32(x).view(np.uint32) != 0x80000000 for x in d)  # no -0 (R8)
    d3, _ = oracle.score(rec_of(agents, now), None, now, hop_scale=3.0)
    assert list(d3[6:8]) == [3.0, 6.0]


def test_remaining_ticks_beyond_2_24_round_to_nearest():
    """R8: D_action = max(0, t_next - now) computed exactly in integers and cast to float32
    round-to-nearest-even ("remaining action duration"; the survey's 2^24 limit is
    replaced by the cast).  Expected values: the exact rational rounded by the textbook rule
    (helpers.round_f32), including the halfway cases 2^24 + 1 (down to even) and 2^24 + 3 (up to
    even), and the largest representable t_next."""
    now = 1000
    rem = [(1 << 24) - 1, 1 << 24, (1 << 24) + 1, (1 << 24) + 2, (1 << 24) + 3, (1 << 25) + 2, (1 << 25) + 6,
           123456789, 0xFFFFFFFF - now]
    d, st = oracle.score(rec_of([dict(d=r) for r in rem], now), None, now)
    assert st == 0
    want = [round_f32(Fraction(r)) for r in rem]
    assert [float(x) for x in d] == [float(x) for x in want]
    assert float(d[2]) == float(1 << 24) and float(d[4]) == float((1 << 24) + 4)
    # now beyond 2^32 (int64 clock): every 32-bit t_next is in the past -> 0
    d, _ = oracle.score(rec_of([dict(d=0), dict(d=5)], 0), None, (1 << 32) + 7)
    assert list(d) == [0.0, 0.0]


def test_bad_records_flagged():
    agents = [dict(cls=3, d=4), dict(cls=tg.CL_INT, d=4, kin=7)]
    d, st = oracle.score(rec_of(agents), np.zeros((1, 4), np.float32), 0)
    assert st & oracle.ST_BAD_RECORD
    assert np.isinf(d[0]) and d[1] == 4.0
    agents = [dict(cls=tg.CL_INT, d=4, kin=0), dict(cls=tg.CL_INT, d=4, kin=1)]
    kin = np.array([[0, 0, np.nan, 0], [1, 0, -1, 0]], np.float32)
    d, st = oracle.score(rec_of(agents), kin, 0)
    assert st & oracle.ST_BAD_KIN
    assert list(d) == [4.0, 4.0]  # the non-finite agent is excluded from the pair scan


# ----------------------------------------------------------------------------------------
# Plan: the paper's worked examples and SPEC examples


def test_prefetch_walkthrough():
    """agent 7 prefetched by replacing inactive resident 5; agent 4 not."""
    g = gold("prefetch_walkthrough.json")
    n = 9
    agents = [dict(phase=tg.PH_IDLE) for _ in range(n)]
    res = np.zeros(n, np.uint8)
    for k, v in g["agents"].items():
        i = int(k)
        agents[i] = dict(d=v["d"]) if v["d"] > 0 else dict(phase=tg.PH_GENERATING)
        res[i] = v["resident"]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, res, np.full(3, g["theta"], np.float32), g["slots"])
    assert sorted(np.nonzero(p["resident"])[0].tolist()) == g["expected_kept"]
    assert p["prefetch"].tolist() == g["expected_prefetch"]
    assert p["evict"].tolist() == g["expected_evict"]
    assert p["status"] == 0


def test_limitation_timeline_evicts_long_action():
    """P:266 / S:242 / S:336: Agent 3 needs space; evict Agent 1 (long action), keep Agent 2."""
    g = gold("limitation_timeline.json")
    agents = [dict(phase=tg.PH_IDLE), dict(d=g["agent1_remaining_action"]),
              dict(d=g["agent2_remaining_action"]), dict(phase=tg.PH_WAITING)]
    res = np.array([0, 1, 1, 0], np.uint8)
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, res, np.zeros(3, np.float32), g["slots"])
    assert p["evict"].tolist() == g["expected_evict"]
    assert sorted(np.nonzero(p["resident"])[0].tolist()) == g["expected_kept"]
    assert p["prefetch"].tolist() == [3]
    # with a threshold, Agent 3 is preloaded while it is still acting
    agents[3] = dict(d=1)
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, res, np.full(3, 4.0, np.float32), g["slots"])
    assert p["prefetch"].tolist() == [3] and p["evict"].tolist() == [1]


def test_spec_dispatch_and_victim_examples():
    # no offloaded agent below threshold -> empty plan
    agents = [dict(d=9), dict(d=12), dict(d=3)]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.array([0, 0, 1], np.uint8), np.full(3, 5.0, np.float32), 10)
    assert p["prefetch"].size == 0 and p["evict"].size == 0
    # budget smaller than the first candidate's footprint -> empty plan, no partial agent
    agents = [dict(d=1, fp=8), dict(d=2, fp=1)]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.zeros(2, np.uint8), np.full(3, 5.0, np.float32), 5)
    assert p["prefetch"].size == 0  # R3: strict prefix stops at the first agent that does not fit
    assert p["cut_bits"] == np.float32(1.0).view(np.uint32) and p["cut_rem"] == 5
    # DistanceMax victims {A1: 30, A2: 5}, need one -> A1
    agents = [dict(phase=tg.PH_WAITING), dict(d=30), dict(d=5)]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.array([0, 1, 1], np.uint8), np.zeros(3, np.float32), 2)
    assert p["evict"].tolist() == [1]
    # every resident is active and the budget is short -> InsufficientMemory
    agents = [dict(phase=tg.PH_GENERATING)] * 3
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.array([1, 1, 0], np.uint8), np.zeros(3, np.float32), 2)
    assert p["status"] & oracle.ST_INSUFFICIENT
    assert p["kept_bytes"] <= 2


def test_equal_distance_tie_reading_R1():
    """S:347 forbids replacing an inactive resident of *equal* distance; reading R1 orders
    by (d, id), so a lower-id candidate outranks an equal-distance resident and a higher-id
    one does not (R1)."""
    agents = [dict(d=4), dict(d=4)]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    p = oracle.plan(rec, d, np.array([0, 1], np.uint8), np.full(3, 10.0, np.float32), 1)
    assert p["prefetch"].tolist() == [0] and p["evict"].tolist() == [1]
    p = oracle.plan(rec, d, np.array([1, 0], np.uint8), np.full(3, 10.0, np.float32), 1)
    assert p["prefetch"].size == 0 and p["evict"].size == 0


# ----------------------------------------------------------------------------------------
# Closed loop with exact next-use distances: canonical trace and Belady's MIN


def run_closed_loop(requests, n_agents, capacity, theta=0.0):
    """requests: list of sets of agents active at each step.  Distances are exact next-use
    distances (steps until the agent is next in a request set; +inf if never).  Returns the
    number of misses (requested agent not resident before the plan)."""
    res = np.zeros(n_agents, np.uint8)
    misses = 0
    T = len(requests)
    for t in range(T):
        agents = []
        for a in range(n_agents):
            nxt = next((u for u in range(t, T) if a in requests[u]), None)
            if nxt is None:
                agents.append(dict(phase=tg.PH_IDLE))
            elif nxt == t:
                agents.append(dict(phase=tg.PH_WAITING))
            else:
                agents.append(dict(d=nxt - t))
        rec = rec_of(agents, now=0)
        d, _ = oracle.score(rec, None, 0)
        misses += sum(1 for a in requests[t] if not res[a])
        p = oracle.plan(rec, d, res, np.full(3, theta, np.float32), capacity)
        res = p["resident"]
        assert all(res[a] for a in requests[t]) or p["status"] & oracle.ST_INSUFFICIENT
    return misses


def lru_misses(trace, capacity):
    cache, misses = [], 0
    for a in trace:
        if a in cache:
            cache.remove(a)
        else:
            misses += 1
            if len(cache) == capacity:
                cache.pop(0)
        cache.append(a)
    return misses


def optimal_misses(requests, capacity):
    """Exhaustive offline optimum: minimum misses over every eviction choice (batched
    requests; the cache must hold each step's request set)."""
    from functools import lru_cache
    T = len(requests)

    @lru_cache(maxsize=None)
    def best(t, cache):
        if t == T:
            return 0
        need = requests[t]
        miss = len(need - cache)
        union = cache | need
        if len(union) <= capacity:
            return miss + best(t + 1, union)
        out = None
        removable = sorted(cache - need)
        k = len(union) - capacity
        for drop in itertools.combinations(removable, k):
            v = best(t + 1, union - frozenset(drop))
            out = v if out is None else min(out, v)
        return miss + out

    return best(0, frozenset())


def test_canonical_trace():
    """S:537 Acceptance 2: 1,2,3,1,2,3 with capacity 2 -> LRU 6, DistanceMax 4 (= optimum)."""
    g = gold("canonical_trace.json")
    reqs = [frozenset([a]) for a in g["trace"]]
    assert lru_misses(g["trace"], g["capacity"]) == g["expected_lru_misses"]
    assert run_closed_loop(reqs, 4, g["capacity"]) == g["expected_distance_misses"]
    assert optimal_misses(reqs, g["capacity"]) == g["expected_distance_misses"]


@pytest.mark.parametrize("batched", [False, True])
def test_belady_equivalence(batched):
    """theta=0, exact distances, uniform sizes -> the planner is Belady's MIN,
    so its misses equal the exhaustive offline optimum, on >= 100 random tiny workloads."""
    rng = np.random.default_rng(1234 + batched)
    for trial in range(120):
        n_agents = int(rng.integers(2, 7))
        cap = int(rng.integers(1, 4))
        T = int(rng.integers(3, 10))
        reqs = []
        for _ in range(T):
            k = int(rng.integers(1, min(cap, n_agents) + 1)) if batched else 1
            reqs.append(frozenset(rng.choice(n_agents, size=k, replace=False).tolist()))
        assert run_closed_loop(reqs, n_agents, cap) == optimal_misses(reqs, cap), (trial, reqs, cap)


# ----------------------------------------------------------------------------------------
# Brute force of the cut on tiny instances (config 1 shape and random sizes)


def brute_force_cut(d, fp, res, theta, cls, budget):
    """Enumerate every subset of agents (all 2^n masks, vectorized); keep the ones that are
    (i) subsets of the eligible agents, (ii) within budget, (iii) closed downward in the
    (d, id) order of the eligible agents, (iv) maximal: the next eligible agent in that
    order does not fit.  Exactly one subset must survive."""
    n = len(d)
    elig = np.array([bool(res[i]) or d[i] == 0 or d[i] < theta[cls[i]] for i in range(n)])
    order = sorted([i for i in range(n) if elig[i]], key=lambda i: (float(d[i]), i))
    masks = np.arange(1 << n, dtype=np.int64)
    bits = ((masks[:, None] >> np.arange(n)) & 1).astype(bool)
    fpv = np.asarray(fp, dtype=np.int64)
    size = bits.astype(np.int64) @ fpv
    ok = ~np.any(bits & ~elig[None, :], axis=1) & (size <= budget)
    k = bits.sum(1)
    prefix = np.zeros(len(order) + 1, dtype=np.int64)  # mask of the first k agents in order
    for j, a in enumerate(order):
        prefix[j + 1] = prefix[j] | (1 << a)
    ok &= masks == prefix[np.minimum(k, len(order))]
    nxt = np.array([fpv[order[j]] if j < len(order) else 0 for j in range(n + 1)])
    ok &= (k >= len(order)) | (size + nxt[np.minimum(k, n)] > budget)
    found = np.nonzero(ok)[0]
    assert len(found) == 1
    return set(np.nonzero(bits[found[0]])[0].tolist()), order


@pytest.mark.parametrize("seed", range(1, 31))
def test_brute_force_config1(seed):
    rng = np.random.default_rng(seed)
    n = 12
    theta = np.array(rng.choice([0.0, 3.0, np.inf], 3), np.float32)
    phase = rng.choice([0, 0, 0, 1, 2, 3], n)
    cls = rng.choice([0, 2], n)
    dd = rng.integers(0, 7, n)
    fp = rng.choice([1, 2, 3, 5], n) if seed % 2 else np.ones(n, int)
    agents = [dict(phase=int(phase[i]), cls=int(cls[i]), d=int(dd[i]), hop=int(dd[i]), fp=int(fp[i])) for i in range(n)]
    rec = rec_of(agents)
    d, _ = oracle.score(rec, None, 0)
    res = (rng.random(n) < 0.4).astype(np.uint8)
    budget = int(rng.integers(0, int(fp.sum()) + 1))
    p = oracle.plan(rec, d, res, theta, budget)
    kept, order = brute_force_cut(d, fp, res, theta, cls, budget)
    assert set(np.nonzero(p["resident"])[0].tolist()) == kept
    pf = [i for i in order if i in kept and not res[i]]
    ev = [i for i in reversed(order) if res[i] and i not in kept]
    assert p["prefetch"].tolist() == pf
    assert p["evict"].tolist() == ev
    assert p["bytes_h2d"] == sum(int(fp[i]) for i in pf)
    zero_out = any(d[i] == 0 and i not in kept for i in range(n))
    assert bool(p["status"] & oracle.ST_INSUFFICIENT) == zero_out


def test_config1_traces_all_variants():
    """Every C1 variant (independent, interaction, diffusion path/star), theta in {0,3,inf},
    seeds 1..20: the closed loop of plans satisfies the brute-force cut at every step."""
    for variant in ("ind", "int", "diff", "diff-star"):
        for th in (0.0, 3.0, np.inf):
            for seed in range(1, 21 if variant == "ind" else 6):
                w = tg.config_c1(seed=seed, theta=(th, th, th), variant=variant)
                res = np.zeros(w.n, np.uint8)
                for s in range(w.steps):
                    kin = w.kin[s] if w.kin is not None else None
                    d, st = oracle.score(w.rec[s], kin, w.now[s], w.hop_scale)
                    p = oracle.plan(w.rec[s], d, res, w.theta, w.budget)
                    cls = (w.rec[s, :, 2] >> 2) & 3
                    kept, _ = brute_force_cut(d, w.rec[s, :, 1], res, w.theta, cls, w.budget)
                    assert set(np.nonzero(p["resident"])[0].tolist()) == kept
                    res = p["resident"]


# ----------------------------------------------------------------------------------------
# LRU baseline as explicit distances (reading R20): pinned to the textbook LRU


def lru_closed_loop(requests, n_agents, capacity):
    """Closed loop of the planner on LRU records (theta = 0): misses = requested agents not
    resident before the plan."""
    res = np.zeros(n_agents, np.uint8)
    last = np.full(n_agents, 0xFFFFFFFF, np.uint32)
    misses = 0
    for t, req in enumerate(requests):
        agents = [dict(phase=tg.PH_WAITING) if a in req else dict(d=1) for a in range(n_agents)]
        rec = oracle.lru_records(rec_of(agents), t, last)
        d, _ = oracle.explicit_dist(rec)
        misses += sum(1 for a in req if not res[a])
        p = oracle.plan(rec, d, res, np.zeros(3, np.float32), capacity)
        res = p["resident"]
    return misses


def test_lru_reading_canonical_trace():
    g = gold("canonical_trace.json")
    reqs = [frozenset([a]) for a in g["trace"]]
    assert lru_closed_loop(reqs, 4, g["capacity"]) == g["expected_lru_misses"]


def test_lru_reading_equals_textbook_lru():
    """Single requests, uniform sizes: the planner on LRU records is LRU (misses equal the
    textbook list-based LRU on random traces)."""
    rng = np.random.default_rng(77)
    for trial in range(150):
        n_agents = int(rng.integers(2, 8))
        cap = int(rng.integers(1, n_agents + 1))
        trace = [int(x) for x in rng.integers(0, n_agents, int(rng.integers(1, 25)))]
        assert lru_closed_loop([frozenset([a]) for a in trace], n_agents, cap) == lru_misses(trace, cap), trial


# ----------------------------------------------------------------------------------------
# Diffusion hop counts (R9): closed forms


def _csr(adj):
    ptr = np.zeros(len(adj) + 1, np.uint64)
    ptr[1:] = np.cumsum([len(a) for a in adj])
    col = np.array([w for a in adj for w in a], np.uint32)
    return ptr, col


def test_bfs_closed_forms():
    # path 0-1-2-...-9 from 0: hop = index; star from the centre: 1; from a leaf: 2
    path = [[i - 1] * (i > 0) + [i + 1] * (i < 9) for i in range(10)]
    assert oracle.bfs_hops(*_csr(path), [0]).tolist() == list(range(10))
    star = [list(range(1, 6))] + [[0]] * 5
    assert oracle.bfs_hops(*_csr(star), [0]).tolist() == [0, 1, 1, 1, 1, 1]
    assert oracle.bfs_hops(*_csr(star), [3]).tolist() == [1, 2, 2, 0, 2, 2]
    # W x H grid graph from the corner: Manhattan distance; two sources: the nearer one
    W, H = 13, 7
    grid = [[] for _ in range(W * H)]
    for y in range(H):
        for x in range(W):
            v = y * W + x
            for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                if 0 <= x + dx < W and 0 <= y + dy < H:
                    grid[v].append((y + dy) * W + x + dx)
    h = oracle.bfs_hops(*_csr(grid), [0])
    assert all(h[y * W + x] == x + y for y in range(H) for x in range(W))
    h2 = oracle.bfs_hops(*_csr(grid), [0, W * H - 1])
    assert all(h2[y * W + x] == min(x + y, (W - 1 - x) + (H - 1 - y)) for y in range(H) for x in range(W))
    # unreachable vertices, out-of-range source ignored
    assert oracle.bfs_hops(*_csr([[1], [0], []]), [0, 99]).tolist() == [0, 1, 0xFFFFFFFF]


def test_prefetch_overlap_plans_two_agents():
    """S:538 / P:174-185: in the two-agent, one-slot timeline the distance planner reloads A at
    step 2 (while B acts, so A's transfer has 5 steps to finish: stall 0), while the reactive
    LRU baseline keeps B and loads A only when A calls again at step 7 (stall = its transfer)."""
    from helpers import two_agent_overlap_records
    F = 1000 * tg.PAGE_BYTES
    recs = two_agent_overlap_records(F)
    res_d = np.zeros(2, np.uint8)
    res_l = np.zeros(2, np.uint8)
    last = np.full(2, 0xFFFFFFFF, np.uint32)
    pf_d, pf_l = {}, {}
    for t in range(len(recs)):
        d, _ = oracle.score(recs[t], None, t)
        p = oracle.plan(recs[t], d, res_d, np.full(3, 10.0, np.float32), F)
        pf_d[t] = list(p["prefetch"])
        res_d = p["resident"]
        rl = oracle.lru_records(recs[t], t, last)
        dl, _ = oracle.explicit_dist(rl)
        q = oracle.plan(rl, dl, res_l, np.zeros(3, np.float32), F)
        pf_l[t] = list(q["prefetch"])
        res_l = q["resident"]
    assert pf_d == {0: [0], 1: [1], 2: [0], 3: [], 4: [], 5: [], 6: [], 7: [], 8: []}
    assert pf_l == {0: [0], 1: [1], 2: [], 3: [], 4: [], 5: [], 6: [], 7: [0], 8: []}


def test_score_sampled_equals_full_score():
    """The sampled oracle (full-size grid parity at 10^6 interaction agents) gives exactly the
    full oracle's distances of the sampled agents (C3 shape, every class)."""
    w = tg.config_c3(seed=4, steps=2, n=6000, budget=10 ** 9)
    rng = np.random.default_rng(1)
    for s in range(2):
        d, st = oracle.score(w.rec[s], w.kin[s], int(w.now[s]), w.hop_scale)
        idx = rng.choice(w.n, 500, replace=False)
        ds, st2 = oracle.score_sampled(w.rec[s], w.kin[s], int(w.now[s]), idx, w.hop_scale)
        assert np.array_equal(ds.view(np.uint32), d[idx].view(np.uint32))
