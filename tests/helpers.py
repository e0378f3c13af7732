"""Small test-only helpers: record construction and exact rational rounding.

No planner arithmetic here — only input construction and textbook numerics used by the
pins (exact round-to-nearest-even of a rational to float32)."""
from fractions import Fraction

import numpy as np

import tracegen as tg


def rec_of(agents, now=0):
    """agents: list of dicts with keys phase, cls, d (remaining ticks / hops), fp, dirty, kin."""
    n = len(agents)
    t_next = np.zeros(n, np.int64)
    for i, a in enumerate(agents):
        if a.get("cls", tg.CL_IND) == tg.CL_DIFF:
            t_next[i] = a.get("hop", 0)
        else:
            t_next[i] = now + a.get("d", 0)
    return tg.pack_records(t_next, [a.get("fp", 1) for a in agents],
                           [a.get("phase", tg.PH_ACTING) for a in agents],
                           [a.get("cls", tg.CL_IND) for a in agents],
                           [a.get("dirty", 0) for a in agents],
                           [a.get("kin", 0) for a in agents])


def round_f32(fr: Fraction) -> np.float32:
    """Correctly rounded (nearest, ties to even) float32 of an exact rational >= 0."""
    if fr == 0:
        return np.float32(0.0)
    approx = np.float32(float(fr))
    cands = {approx, np.nextafter(approx, np.float32(np.inf)), np.nextafter(approx, np.float32(0))}
    best = None
    for c in cands:
        if not np.isfinite(c):
            continue
        err = abs(Fraction(float(c)) - fr)
        key = (err, int(np.float32(c).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def keys_of(d, ids):
    return (np.asarray(d, np.float32).view(np.uint32).astype(np.uint64) << np.uint64(32)) | \
        np.asarray(ids, np.uint64)


def two_agent_overlap_records(F):
    """SPEC acceptance #3 / P:174-185 timeline: agents A (0) and B (1), one slot.  A
    calls the LLM at step 0, acts until step 7; B calls at step 1 and then acts for 19 steps,
    longer than A's transfer: the distance policy reloads A while B acts."""
    recs = []
    for t in range(9):
        if t == 0:
            ag = [dict(phase=tg.PH_WAITING), dict(d=1)]
        elif t == 1:
            ag = [dict(d=6), dict(phase=tg.PH_WAITING)]
        elif t < 7:
            ag = [dict(d=7 - t), dict(d=20 - t)]
        elif t == 7:
            ag = [dict(phase=tg.PH_WAITING), dict(d=20 - t)]
        else:
            ag = [dict(phase=tg.PH_GENERATING), dict(d=20 - t)]
        for a in ag:
            a["fp"] = F
        recs.append(rec_of(ag, now=t))
    return np.stack(recs)
