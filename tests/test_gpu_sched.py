"""GPU parity of the preemptive load scheduler (scalesim_sched_run, NEXT #2) against the
oracle (oracle/sched.py): the slot trace (which task's which chunk moved when), the task
table (states, chunks done, coalesced priorities, preemptions, finish slots) bit-exact, and
the bytes: every finished task's device region equals its host source, a cancelled task's
moved chunks too.  The paper's preemption example, coalescing, stale cancellation, idle
slots, ragged chunk tails, and 300 randomized schedules (acceptance #8's generator)."""
import numpy as np
import pytest

from oracle import sched as S

pytestmark = pytest.mark.gpu

CH = 1 << 16
REGION = 8 * CH


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


@pytest.fixture(scope="module")
def arenas():
    import torch
    from gpu_harness import fill_pattern
    n_agents = 16
    host = torch.empty(n_agents * REGION, dtype=torch.uint8, pin_memory=True)
    fill_pattern(host)
    dev = torch.zeros(n_agents * REGION, dtype=torch.uint8, device="cuda")
    return host, dev, n_agents


def to_events(evs):
    from paper_2601_21473_b200.planner import LOAD_EVENT
    a = np.zeros(len(evs), LOAD_EVENT)
    for i, e in enumerate(evs):
        a[i] = (e["slot"], e["kind"], e["agent"], e["priority"], e["agent"] * REGION, e["agent"] * REGION, e["bytes"])
    return a


def check(evs, threshold, arenas, max_slots=10_000):
    import torch
    from paper_2601_21473_b200.planner import sched_run
    host, dev, n_agents = arenas
    dev.zero_()
    tr, tk, n = sched_run(to_events(evs), n_agents, threshold, CH, host, dev, max_slots)
    # the oracle sees the same float32 priorities
    evs32 = [dict(e, priority=float(np.float32(e["priority"]))) for e in evs]
    o = S.run(evs32, float(np.float32(threshold)), CH, max_slots)
    assert n == o["n_slots"] and [tuple(int(x) for x in r) for r in tr] == o["trace"], (tr[:10], o["trace"][:10])
    assert len(tk) == len(o["tasks"])
    for g, t in zip(tk, o["tasks"]):
        assert (g["agent"], g["chunks"], g["done"], g["state"], g["preemptions"]) == \
            (t["agent"], t["chunks"], t["done"], t["state"], t["preemptions"]), (g, t)
        assert np.float32(g["priority"]) == np.float32(t["priority"])
        assert g["finish_slot"] == (0xFFFFFFFF if t["finish_slot"] is None else t["finish_slot"])
    torch.cuda.synchronize()
    hd, dd = host.numpy(), dev.cpu().numpy()
    for t in o["tasks"]:
        a = t["agent"]
        moved = min(t["bytes"], t["done"] * CH)
        assert np.array_equal(dd[a * REGION:a * REGION + moved], hd[a * REGION:a * REGION + moved]), t
    return o


def ev(slot, agent, prio, nbytes=CH, kind=S.SUBMIT):
    return dict(slot=slot, kind=kind, agent=agent, priority=float(prio), bytes=nbytes)


def test_paper_example_and_spec_cases(arenas):
    o = check([ev(0, 7, 2.0, 3 * CH), ev(1, 9, 0.0, 2 * CH)], 4.0, arenas)
    assert o["trace"] == [(0, 0), (1, 0), (1, 1), (0, 1), (0, 2)]
    check([ev(3, 1, 5.0, CH)], 9.0, arenas)                                               # idle start
    check([ev(0, 1, 3.0, 3 * CH), ev(1, 2, 3.0, CH)], 9.0, arenas)                         # ties
    check([ev(0, 3, 2.0, 2 * CH), ev(0, 4, 5.0, 2 * CH), ev(1, 4, 1.0, 2 * CH)], 9.0, arenas)  # coalescing
    check([ev(0, 1, 1.0, 3 * CH), ev(0, 2, 2.0, CH), ev(1, 2, 7.0, kind=S.CANCEL), ev(1, 1, 9.0, kind=S.CANCEL),
           ev(4, 2, 3.0, CH)], 7.0, arenas)                                                # cancellation
    check([ev(0, 5, 1.0, 3 * CH + 48), ev(0, 6, 0.5, 17)], 9.0, arenas)                    # ragged tails
    check([], 9.0, arenas)                                                                 # nothing to do


def test_randomized_schedules(arenas):
    rng = np.random.default_rng(20)
    pre = 0
    for sc in range(300):
        n_ev = int(rng.integers(1, 30))
        evs = []
        sizes = rng.integers(1, 6 * CH, 16) // 16 * 16 + 16
        for _ in range(n_ev):
            kind = S.CANCEL if rng.random() < 0.15 else S.SUBMIT
            prio = float(rng.choice([0.0, 1.0, 2.0, 5.0]) if rng.random() < 0.7 else rng.uniform(0, 10))
            a = int(rng.integers(0, 16))
            evs.append(dict(slot=int(rng.integers(0, 40)), kind=kind, agent=a, priority=prio, bytes=int(sizes[a])))
        evs.sort(key=lambda e: e["slot"])
        o = check(evs, float(rng.choice([4.0, 100.0])), arenas)
        pre += sum(t["preemptions"] for t in o["tasks"])
    assert pre > 50
