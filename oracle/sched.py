"""CPU oracle of the preemptive priority load scheduler (NEXT #2).

TEST INFRASTRUCTURE ONLY: only tests/ and bench.py's cpu/reference legs may import this
module; the product (paper_2601_21473_b200/, include/scalesim.h) never does, and this module
imports nothing from the product.  Plain Python loops over small event lists.

What it computes (App. A "Load task scheduler" / "Preemption support", P:483-491;
SPEC.md S:291-293 design decisions, S:324-327 LoadTask, S:348-356 scheduler_submit, S:366-374
cancel_stale_tasks; readings R21-R23 in DESIGN.md §3):

  * one channel: at most one task transfers at a time ("one active LoadTask");
  * a task moves its bytes in chunks of `chunk_bytes` (default 16 MB), one chunk per
    slot; the scheduler decides only at chunk boundaries ("preemption checks only at
    chunk boundaries");
  * priority = invocation distance, lower = more urgent, ties by ascending task id (S:351,
    S:356 "two tasks, equal priority -> lower task id first");
  * a submission whose priority is strictly lower than the executing task's preempts it at
    the next boundary: the executing task is re-enqueued (Preempted) and resumes later with
    its completed chunks kept ("interrupts the ongoing task, re-enqueues it back into the
    queue, and inserts the urgent task at the front"; S:292 resume keeps chunks);
  * a submission for an agent that already has an active (queued, preempted or executing)
    task is coalesced into it: the task's priority becomes the minimum of the two and no task
    is created (S:351 errors clause);
  * cancel_stale: a queued or preempted task whose agent's refreshed distance is >= the
    prefetch threshold is cancelled; the executing task never is (R22: ">= theta"
    = no longer eligible under R4's strict d < theta).

Event model (R23): events carry the slot before which they are admitted; at each boundary k
the events with slot <= k are applied in their order, then the task to run slot k is chosen,
then one chunk of it moves.  A slot with no runnable task is idle.  The trace lists, per
slot, (task id, chunk index) or (IDLE, 0).
"""
from __future__ import annotations

SUBMIT, CANCEL = 0, 1
QUEUED, EXECUTING, PREEMPTED, DONE, CANCELLED = 0, 1, 2, 3, 4
IDLE = 0xFFFFFFFF


def n_chunks(nbytes: int, chunk_bytes: int) -> int:
    return max(1, (nbytes + chunk_bytes - 1) // chunk_bytes)


def run(events, threshold: float, chunk_bytes: int, max_slots: int):
    """events: list of dicts {slot, kind, agent, priority, bytes} sorted by slot (stable).
    Returns dict(trace=[(task, chunk)], tasks=[dict(agent, priority, chunks, done, state,
    preemptions, finish_slot)], n_slots)."""
    tasks = []
    active = {}          # agent -> task id (queued / preempted / executing)
    executing = None
    trace = []
    ev = 0
    slot = 0
    while slot < max_slots:
        # (1) admit this boundary's events, in order
        while ev < len(events) and events[ev]["slot"] <= slot:
            e = events[ev]
            ev += 1
            a = e["agent"]
            if e["kind"] == SUBMIT:
                t = active.get(a)
                if t is not None:  # coalesce: the minimum of the two priorities
                    tasks[t]["priority"] = min(tasks[t]["priority"], e["priority"])
                else:
                    tasks.append(dict(agent=a, priority=e["priority"], chunks=n_chunks(e["bytes"], chunk_bytes),
                                      bytes=e["bytes"], done=0, state=QUEUED, preemptions=0, finish_slot=None,
                                      submit_slot=e["slot"]))
                    active[a] = len(tasks) - 1
            else:  # refreshed distance: cancel a waiting task that is no longer eligible
                t = active.get(a)
                if t is not None and tasks[t]["state"] in (QUEUED, PREEMPTED) and e["priority"] >= threshold:
                    tasks[t]["state"] = CANCELLED
                    del active[a]
        # (2) choose the task of this slot
        waiting = [i for i, t in enumerate(tasks) if t["state"] in (QUEUED, PREEMPTED)]
        best = min(waiting, key=lambda i: (tasks[i]["priority"], i)) if waiting else None
        if executing is None:
            if best is not None:
                executing = best
                tasks[best]["state"] = EXECUTING
        elif best is not None and tasks[best]["priority"] < tasks[executing]["priority"]:
            tasks[executing]["state"] = PREEMPTED
            tasks[executing]["preemptions"] += 1
            executing = best
            tasks[best]["state"] = EXECUTING
        if executing is None:
            if ev >= len(events):
                break
            trace.append((IDLE, 0))
            slot += 1
            continue
        # (3) one chunk of the executing task
        t = tasks[executing]
        trace.append((executing, t["done"]))
        t["done"] += 1
        if t["done"] == t["chunks"]:
            t["state"] = DONE
            t["finish_slot"] = slot
            del active[t["agent"]]
            executing = None
        slot += 1
    return dict(trace=trace, tasks=tasks, n_slots=len(trace))
