"""Pins of the scheduler oracle (oracle/sched.py, NEXT #2) against the paper's and SPEC's
examples and invariants, checked from the trace by independent bookkeeping:

- P:489 / S:354: a D=2 transfer is interrupted when an urgent D=0 task arrives, re-enqueued,
  and resumes with its completed chunks after the urgent one (Figure "preemption").
- S:355: an empty queue and an idle channel: a task starts at the next boundary.
- S:356: equal priority: the lower task id first (no preemption on ties).
- S:351: a duplicate submission for an agent is coalesced (minimum priority, no new task).
- S:368-373: a waiting task whose agent's distance reaches the threshold is cancelled; the
  executing task never is; a later submission for that agent is a new task.
- S:543 acceptance #8 over 600 randomized schedules: no task lost, priority(executing) <=
  priority(every waiting task) at every boundary, each finished task moves exactly its chunks
  once each and in order (resumed tasks only their remaining chunks).
"""
import numpy as np

from oracle import sched as S

CH = 1 << 20


def ev(slot, agent, prio, nbytes=CH, kind=S.SUBMIT):
    return dict(slot=slot, kind=kind, agent=agent, priority=float(prio), bytes=nbytes)


def test_paper_preemption_example():
    # t=0: D=2 task executing; t=1: urgent D=0 task arrives -> D=2 interrupted, D=0 runs
    out = S.run([ev(0, 7, 2.0, 3 * CH), ev(1, 9, 0.0, 2 * CH)], threshold=4.0, chunk_bytes=CH, max_slots=100)
    assert out["trace"] == [(0, 0), (1, 0), (1, 1), (0, 1), (0, 2)]
    assert out["tasks"][0]["preemptions"] == 1 and out["tasks"][1]["preemptions"] == 0
    assert [t["state"] for t in out["tasks"]] == [S.DONE, S.DONE]


def test_idle_channel_starts_at_next_boundary():
    out = S.run([ev(3, 1, 5.0, CH)], threshold=9.0, chunk_bytes=CH, max_slots=100)
    assert out["trace"] == [(S.IDLE, 0)] * 3 + [(0, 0)]


def test_equal_priority_lower_id_first_and_no_preemption_on_ties():
    out = S.run([ev(0, 1, 3.0, 2 * CH), ev(0, 2, 3.0, 2 * CH)], 9.0, CH, 100)
    assert out["trace"] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    # a tie arriving while the first task runs does not interrupt it
    out = S.run([ev(0, 1, 3.0, 3 * CH), ev(1, 2, 3.0, CH)], 9.0, CH, 100)
    assert out["trace"] == [(0, 0), (0, 1), (0, 2), (1, 0)]


def test_coalescing_duplicate_submissions():
    # agent 4's second submission (more urgent) is merged: no task 2, task 1 jumps ahead
    out = S.run([ev(0, 3, 2.0, 2 * CH), ev(0, 4, 5.0, 2 * CH), ev(1, 4, 1.0, 2 * CH)], 9.0, CH, 100)
    assert len(out["tasks"]) == 2 and out["tasks"][1]["priority"] == 1.0
    assert out["trace"] == [(0, 0), (1, 0), (1, 1), (0, 1)]
    # a less urgent duplicate does not raise the priority
    out = S.run([ev(0, 3, 2.0, CH), ev(0, 3, 6.0, CH)], 9.0, CH, 100)
    assert len(out["tasks"]) == 1 and out["tasks"][0]["priority"] == 2.0


def test_cancel_stale_waiting_tasks_only():
    evs = [ev(0, 1, 1.0, 3 * CH), ev(0, 2, 2.0, CH),
           ev(1, 2, 7.0, kind=S.CANCEL),   # waiting task of agent 2: distance rose to theta -> cancelled
           ev(1, 1, 9.0, kind=S.CANCEL),   # agent 1 is executing: never cancelled
           ev(4, 2, 3.0, CH)]              # a new submission for agent 2: a new task
    out = S.run(evs, threshold=7.0, chunk_bytes=CH, max_slots=100)
    st = [t["state"] for t in out["tasks"]]
    assert st == [S.DONE, S.CANCELLED, S.DONE]
    assert out["trace"] == [(0, 0), (0, 1), (0, 2), (S.IDLE, 0), (2, 0)]
    # below the threshold: kept
    out = S.run([ev(0, 1, 1.0, 2 * CH), ev(0, 2, 2.0, CH), ev(1, 2, 6.9, kind=S.CANCEL)], 7.0, CH, 100)
    assert [t["state"] for t in out["tasks"]] == [S.DONE, S.DONE]


def random_events(rng, n_ev, n_agents, max_slot):
    evs = []
    for _ in range(n_ev):
        kind = S.CANCEL if rng.random() < 0.15 else S.SUBMIT
        prio = float(rng.choice([0.0, 1.0, 2.0, 3.0, 5.0, 8.0]) if rng.random() < 0.7 else rng.uniform(0, 10))
        evs.append(dict(slot=int(rng.integers(0, max_slot)), kind=kind, agent=int(rng.integers(0, n_agents)),
                        priority=prio, bytes=int(rng.integers(1, 6 * CH))))
    evs.sort(key=lambda e: e["slot"])  # (stable: same-slot events keep their order)
    return evs


def check_schedule(evs, out, threshold):
    """Acceptance #8 from the events and the trace, with bookkeeping of its own."""
    trace, tasks = out["trace"], out["tasks"]
    # task creation replayed: a submission creates a task iff its agent has no live task
    live, created = {}, []
    finish = {}
    for i, (t, k) in enumerate(trace):
        if t != S.IDLE and k + 1 == tasks[t]["chunks"]:
            finish[t] = i
    prio = {}
    cancelled_at = {}
    ev_i = 0
    for slot in range(len(trace) + 1):
        while ev_i < len(evs) and evs[ev_i]["slot"] <= slot:
            e = evs[ev_i]
            ev_i += 1
            a = e["agent"]
            t = live.get(a)
            if t is not None and (t in finish and finish[t] < slot):
                del live[a]
                t = None
            if e["kind"] == S.SUBMIT:
                if t is None:
                    created.append(a)
                    live[a] = len(created) - 1
                    prio[len(created) - 1] = e["priority"]
                else:
                    prio[t] = min(prio[t], e["priority"])
            elif t is not None and e["priority"] >= threshold:
                running = slot > 0 and trace[slot - 1][0] == t and trace[slot - 1][1] + 1 < tasks[t]["chunks"]
                if not running:
                    cancelled_at[t] = slot
                    del live[a]
        if slot == len(trace):
            break
        t, k = trace[slot]
        if t == S.IDLE:  # idle only when nothing is waiting
            assert all(u in finish and finish[u] < slot for u in live.values()), (slot, live)
            continue
        # (b) priority invariant: the running task is at least as urgent as every waiting one
        for u in live.values():
            if u != t and not (u in finish and finish[u] < slot):
                assert prio[t] <= prio[u], (slot, t, u, prio[t], prio[u])
    assert len(created) == len(tasks)
    assert [tk["agent"] for tk in tasks] == created
    # (a) no task lost, (c) each finished task's chunks exactly once, in order
    per = {}
    for t, k in trace:
        if t != S.IDLE:
            per.setdefault(t, []).append(k)
    for i, tk in enumerate(tasks):
        if tk["state"] == S.DONE:
            assert per.get(i) == list(range(tk["chunks"])), (i, per.get(i))
        else:
            assert tk["state"] == S.CANCELLED and i in cancelled_at, (i, tk)
            assert per.get(i, []) == list(range(len(per.get(i, []))))  # a prefix moved before it was cancelled
    assert sum(len(v) for v in per.values()) == sum(1 for t, _ in trace if t != S.IDLE)


def test_acceptance_8_randomized_schedules():
    rng = np.random.default_rng(8)
    n_pre = 0
    for sc in range(600):
        evs = random_events(rng, int(rng.integers(1, 40)), int(rng.integers(1, 12)), int(rng.integers(1, 60)))
        theta = float(rng.choice([4.0, 6.0, 100.0]))
        out = S.run(evs, theta, CH, 100_000)
        assert all(t["state"] in (S.DONE, S.CANCELLED) for t in out["tasks"]), sc
        check_schedule(evs, out, theta)
        n_pre += sum(t["preemptions"] for t in out["tasks"])
    assert n_pre > 100  # the schedules exercise preemption
