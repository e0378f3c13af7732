"""Synthetic AgentSociety-shaped traces for the three workload classes.

Everything is seeded (numpy PCG64) and step-quantized: 1 tick = 1 simulation step (R15).
The output of every generator is the per-step agent state the simulation frontend
hands to the planner: phase, action-end tick or remaining hop count, dirty bit, and for
interaction agents their kinematics.  No distance is computed here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PH_ACTING, PH_WAITING, PH_GENERATING, PH_IDLE = 0, 1, 2, 3
CL_IND, CL_INT, CL_DIFF = 0, 1, 2
KIND_LORA, KIND_KV, KIND_HIST = 0, 1, 2
PAGE_BYTES = 65536
UNREACHABLE = 0xFFFFFFFF

# Block sizes (bytes).  LoRA rank 16 over the public Qwen2.5 configs:
#   7B q/k/v/o x 28 layers = 20,185,088 B;  0.5B q/v x 24 layers = 2,162,688 B.
# KV page = 16 tokens x KV bytes/token: 7B 917,504 B; 0.5B 196,608 B.  HIST 64 KiB.
LORA_7B, KV_7B = 20_185_088, 917_504
LORA_05B, KV_05B, HIST = 2_162_688, 196_608, 65_536


def pack_records(t_next, footprint, phase, cls, dirty, kin_idx) -> np.ndarray:
    """Pack per-agent state into the 16-byte record (n, 4) uint32."""
    n = len(phase)
    rec = np.empty((n, 4), dtype=np.uint32)
    rec[:, 0] = np.asarray(t_next, dtype=np.uint64).astype(np.uint32)
    rec[:, 1] = np.asarray(footprint, dtype=np.uint32)
    rec[:, 2] = (np.asarray(phase, dtype=np.uint32) & 3) | ((np.asarray(cls, dtype=np.uint32) & 3) << 2) \
        | ((np.asarray(dirty, dtype=np.uint32) & 1) << 4)
    rec[:, 3] = np.asarray(kin_idx, dtype=np.uint32)
    return rec


@dataclass
class Blocks:
    """CSR agent -> blocks.  Sizes are multiples of PAGE_BYTES."""
    blk_ptr: np.ndarray  # (n+1,) uint64
    blk_size: np.ndarray  # (nb,) uint32
    blk_host_off: np.ndarray  # (nb,) uint64
    blk_kind: np.ndarray  # (nb,) uint8
    host_bytes: int  # size of the pinned host arena the offsets index

    @property
    def footprint(self) -> np.ndarray:
        n = len(self.blk_ptr) - 1
        agent = np.repeat(np.arange(n), np.diff(self.blk_ptr).astype(np.int64))
        fp = np.zeros(n, dtype=np.uint64)
        np.add.at(fp, agent, self.blk_size.astype(np.uint64))
        return fp


def make_blocks(kinds_per_agent, sizes_per_agent, host_bytes: Optional[int] = None,
                page_bytes: int = PAGE_BYTES) -> Blocks:
    """Build the CSR block table.  Host offsets are laid out contiguously; when the total
    exceeds ``host_bytes`` they alias modulo the arena (bytes moved are still real)."""
    counts = np.array([len(k) for k in kinds_per_agent], dtype=np.uint64)
    blk_ptr = np.zeros(len(counts) + 1, dtype=np.uint64)
    blk_ptr[1:] = np.cumsum(counts)
    blk_kind = np.concatenate([np.asarray(k, np.uint8) for k in kinds_per_agent]) if len(counts) else \
        np.zeros(0, np.uint8)
    blk_size = np.concatenate([np.asarray(s, np.uint32) for s in sizes_per_agent]) if len(counts) else \
        np.zeros(0, np.uint32)
    assert np.all(blk_size % page_bytes == 0)
    off = np.zeros(len(blk_size), dtype=np.uint64)
    if len(blk_size):
        off[1:] = np.cumsum(blk_size.astype(np.uint64))[:-1]
    total = int(blk_size.astype(np.uint64).sum())
    if host_bytes is None:
        host_bytes = max(total, page_bytes)
    if total > host_bytes:
        # alias: keep each block inside the arena
        hb = host_bytes // page_bytes * page_bytes
        off = off % np.uint64(hb)
        over = off + blk_size.astype(np.uint64) > np.uint64(hb)
        off[over] = 0
    return Blocks(blk_ptr, blk_size, off, blk_kind, int(host_bytes))


def _blocks_vectorized(n, lora, kv, n_kv, hist, host_bytes):
    """Fast path of make_blocks for [LoRA, KV x n_kv[i], (HIST)] per agent."""
    per = 1 + n_kv.astype(np.int64) + (1 if hist else 0)
    blk_ptr = np.zeros(n + 1, np.uint64)
    blk_ptr[1:] = np.cumsum(per)
    nb = int(blk_ptr[-1])
    kind = np.full(nb, KIND_KV, np.uint8)
    size = np.full(nb, kv, np.uint32)
    starts = blk_ptr[:-1].astype(np.int64)
    kind[starts] = KIND_LORA
    size[starts] = lora
    if hist:
        last = blk_ptr[1:].astype(np.int64) - 1
        kind[last] = KIND_HIST
        size[last] = hist
    off = np.zeros(nb, np.uint64)
    if nb:
        off[1:] = np.cumsum(size.astype(np.uint64))[:-1]
    total = int(size.astype(np.uint64).sum())
    if host_bytes is None:
        host_bytes = total
    if total > host_bytes:
        hb = np.uint64(host_bytes // PAGE_BYTES * PAGE_BYTES)
        off = off % hb
        over = off + size.astype(np.uint64) > hb
        off[over] = 0
    return Blocks(blk_ptr, size, off, kind, int(host_bytes))


@dataclass
class Workload:
    name: str
    n: int
    now: np.ndarray  # (steps,) int64: tick of each step
    rec: np.ndarray  # (steps, n, 4) uint32
    kin: Optional[np.ndarray]  # (steps, n_kin, 4) float32 or None
    blocks: Blocks
    budget: int
    theta: np.ndarray  # (3,) float32
    hop_scale: float = 1.0
    page_bytes: int = PAGE_BYTES
    meta: dict = field(default_factory=dict)

    @property
    def steps(self) -> int:
        return int(self.rec.shape[0])

    @property
    def n_kin(self) -> int:
        return 0 if self.kin is None else int(self.kin.shape[1])

    @property
    def footprint(self) -> np.ndarray:
        return self.rec[0, :, 1].astype(np.uint64)


# ------------------------------------------------------------------------------------
# Lifecycle simulators.  Each returns per-step (phase, t_next, dirty) arrays.


def _calibrate_mu0(rng, active: float, sigma: float, g_mean: float) -> float:
    """Mean action duration scale mu0 so that mean_i g/(g+mu_i) ~= active."""
    z = rng.standard_normal(20000)
    lo, hi = 1.0, 1e6
    for _ in range(100):
        mid = np.sqrt(lo * hi)
        mu = np.maximum(1.0, mid * np.exp(sigma * z))
        frac = np.mean(g_mean / (g_mean + mu))
        if frac > active:
            lo = mid
        else:
            hi = mid
    return float(np.sqrt(lo * hi))


def gen_independent(n: int, steps: int, seed: int, active: float = 0.05, sigma: float = 1.0,
                    g_choices=(1, 2, 3), fixed_dur: Optional[tuple] = None, t0: int = 0,
                    dirty_window: int = 16, noise: float = 0.0):
    """AgentSociety-shaped independent agents.

    Each agent alternates an LLM phase of g ~ U(g_choices) steps (first step WAITING, then
    GENERATING) and an action of integer duration ~ Geometric(1/mu_i), mu_i ~
    LogNormal(ln mu0, sigma) (skewed invocation orders, heavy integer ties).  With
    ``fixed_dur=(lo, hi)`` durations are U{lo..hi} instead.  Initial phases are staggered.
    ``noise`` > 0: the recorded action end is an estimate ("an optional
    multiplicative noise knob perturbs D_action to model imperfect estimates"; "these
    estimates do not need to be exact"): each action's duration is reported as
    max(1, round(true duration * exp(noise * z))), z ~ N(0, 1) drawn once per action, while the
    agent's phases follow the true durations (noise = 0: exact, and no extra random draws).
    Returns phase, t_next, dirty arrays of shape (steps, n)."""
    nz_rng = np.random.Generator(np.random.PCG64(seed + 7919)) if noise > 0 else None

    def estimate(start, dur):
        if nz_rng is None:
            return start + dur
        z = nz_rng.standard_normal(len(dur))
        return start + np.maximum(1, np.rint(dur * np.exp(noise * z))).astype(np.int64)
    rng = np.random.Generator(np.random.PCG64(seed))
    g_choices = np.asarray(g_choices, dtype=np.int64)
    if fixed_dur is None:
        mu0 = _calibrate_mu0(rng, active, sigma, float(g_choices.mean()))
        mu = np.maximum(1.0, mu0 * np.exp(sigma * rng.standard_normal(n)))

        def draw_dur(idx):
            return rng.geometric(1.0 / mu[idx]).astype(np.int64)
    else:
        lo, hi = fixed_dur
        mu = np.full(n, (lo + hi) / 2.0)

        def draw_dur(idx):
            return rng.integers(lo, hi + 1, size=len(idx)).astype(np.int64)

    # staggered start: generating with prob g/(g+mu), else acting part-way through
    gm = float(g_choices.mean())
    gen_now = rng.random(n) < gm / (gm + mu)
    phase = np.where(gen_now, PH_GENERATING, PH_ACTING).astype(np.int64)
    all_idx = np.arange(n)
    dur = draw_dur(all_idx)
    if fixed_dur is None:
        remain = dur  # geometric durations are memoryless: residual life ~ same law
    else:
        remain = 1 + (rng.random(n) * dur).astype(np.int64)
    t_end = np.where(gen_now, t0 + rng.choice(g_choices, size=n), t0 + remain)
    est_end = estimate(np.full(n, t0, np.int64), remain)  # (used while ACTING)
    last_gen = np.where(gen_now, t0, -(10 ** 9))
    gen_start = np.where(gen_now, t0 - 1, -(10 ** 9))

    P = np.empty((steps, n), np.uint8)
    T = np.empty((steps, n), np.int64)
    D = np.empty((steps, n), np.uint8)
    for s in range(steps):
        t = t0 + s
        # LLM phase finished -> start a new action
        done_gen = (phase != PH_ACTING) & (t_end <= t)
        idx = np.nonzero(done_gen)[0]
        if len(idx):
            phase[idx] = PH_ACTING
            dd = draw_dur(idx)
            t_end[idx] = t + dd
            est_end[idx] = estimate(np.full(len(idx), t, np.int64), dd)
        # action finished -> issue an LLM call (S:146 activations at t_end)
        done_act = (phase == PH_ACTING) & (t_end <= t)
        idx = np.nonzero(done_act)[0]
        if len(idx):
            phase[idx] = PH_WAITING
            gen_start[idx] = t
            t_end[idx] = t + rng.choice(g_choices, size=len(idx))
        waiting = (phase == PH_WAITING) & (gen_start < t)
        phase[waiting] = PH_GENERATING
        act = phase != PH_ACTING
        last_gen[act] = t
        P[s] = phase
        T[s] = np.where(phase == PH_ACTING, est_end, 0)
        D[s] = (t - last_gen) < dirty_window
    return P, T, D


def _reflect(x, v, L):
    x = x + v
    lo = x < 0
    x[lo] = -x[lo]
    v[lo] = -v[lo]
    hi = x > L
    x[hi] = 2 * L - x[hi]
    v[hi] = -v[hi]
    return x, v


def gen_interaction(n: int, steps: int, seed: int, active: float = 0.05, arena: float = 2000.0,
                    r_int: float = 1.0, v_max: float = 1.0, sigma: float = 1.0,
                    g_choices=(1, 2, 3), t0: int = 0, dirty_window: int = 16):
    """Generative-Agents-style spatial agents.

    Agents run the independent lifecycle, and move with constant velocity (speed
    U[0, v_max], uniform heading) in an arena x arena square with reflecting walls.  When
    two ACTING agents come within r_int, both end their action and issue an LLM call; an
    agent that interacted cannot trigger again until its next action ends (cooldown,
    S:188).  Returns phase, t_next, dirty (steps, n) and kin (steps, n, 4) float32."""
    from scipy.spatial import cKDTree

    rng = np.random.Generator(np.random.PCG64(seed))
    g_choices = np.asarray(g_choices, dtype=np.int64)
    mu0 = _calibrate_mu0(rng, active, sigma, float(g_choices.mean()))
    mu = np.maximum(1.0, mu0 * np.exp(sigma * rng.standard_normal(n)))
    gm = float(g_choices.mean())
    gen_now = rng.random(n) < gm / (gm + mu)
    phase = np.where(gen_now, PH_GENERATING, PH_ACTING).astype(np.int64)
    dur = rng.geometric(1.0 / mu).astype(np.int64)
    t_end = np.where(gen_now, t0 + rng.choice(g_choices, size=n), t0 + dur)
    gen_start = np.where(gen_now, t0 - 1, -(10 ** 9))
    last_gen = np.where(gen_now, t0, -(10 ** 9))
    cooldown = np.zeros(n, bool)
    pos = rng.random((n, 2)) * arena
    speed = rng.random(n) * v_max
    head = rng.random(n) * 2 * np.pi
    vel = np.stack([speed * np.cos(head), speed * np.sin(head)], axis=1)

    P = np.empty((steps, n), np.uint8)
    T = np.empty((steps, n), np.int64)
    D = np.empty((steps, n), np.uint8)
    K = np.empty((steps, n, 4), np.float32)
    for s in range(steps):
        t = t0 + s
        if s > 0:
            for c in range(2):
                pos[:, c], vel[:, c] = _reflect(pos[:, c], vel[:, c], arena)
        done_gen = (phase != PH_ACTING) & (t_end <= t)
        idx = np.nonzero(done_gen)[0]
        if len(idx):
            phase[idx] = PH_ACTING
            t_end[idx] = t + rng.geometric(1.0 / mu[idx]).astype(np.int64)
        done_act = (phase == PH_ACTING) & (t_end <= t)
        cooldown[done_act] = False
        # spatial interactions among ACTING agents not in cooldown
        cand = np.nonzero((phase == PH_ACTING) & ~cooldown & ~done_act)[0]
        trig = np.zeros(n, bool)
        if len(cand) > 1:
            pairs = cKDTree(pos[cand]).query_pairs(r_int, output_type="ndarray")
            if len(pairs):
                trig[cand[pairs[:, 0]]] = True
                trig[cand[pairs[:, 1]]] = True
        cooldown |= trig
        start = done_act | trig
        idx = np.nonzero(start)[0]
        if len(idx):
            phase[idx] = PH_WAITING
            gen_start[idx] = t
            t_end[idx] = t + rng.choice(g_choices, size=len(idx))
        waiting = (phase == PH_WAITING) & (gen_start < t)
        phase[waiting] = PH_GENERATING
        act = phase != PH_ACTING
        last_gen[act] = t
        P[s] = phase
        T[s] = np.where(phase == PH_ACTING, t_end, 0)
        D[s] = (t - last_gen) < dirty_window
        K[s, :, 0:2] = pos
        K[s, :, 2:4] = vel
    return P, T, D, K


def ba_graph(n: int, m: int, seed: int):
    """Barabási–Albert preferential attachment graph (social-network-like), adjacency list."""
    rng = np.random.Generator(np.random.PCG64(seed))
    m0 = max(m, 1)
    adj = [[] for _ in range(n)]
    # start from a clique of m0+1 nodes
    targets_pool = []
    init = min(n, m0 + 1)
    for i in range(init):
        for j in range(i + 1, init):
            adj[i].append(j)
            adj[j].append(i)
            targets_pool += [i, j]
    pool = np.empty(2 * m0 * n + len(targets_pool) + 8, dtype=np.int64)
    pool[:len(targets_pool)] = targets_pool
    plen = len(targets_pool)
    for v in range(init, n):
        chosen = set()
        while len(chosen) < min(m0, v):
            u = int(pool[rng.integers(0, plen)]) if plen else int(rng.integers(0, v))
            chosen.add(u)
        for u in sorted(chosen):
            adj[v].append(u)
            adj[u].append(v)
            pool[plen] = u
            pool[plen + 1] = v
            plen += 2
    return adj


def bfs_hops(adj, sources):
    """Breadth-first hop count from the source set; UNREACHABLE where not reachable."""
    n = len(adj)
    hop = np.full(n, UNREACHABLE, dtype=np.int64)
    frontier = list(dict.fromkeys(int(s) for s in sources))
    for s in frontier:
        hop[s] = 0
    level = 0
    while frontier:
        nxt = []
        for u in frontier:
            for w in adj[u]:
                if hop[w] == UNREACHABLE:
                    hop[w] = level + 1
                    nxt.append(w)
        frontier = nxt
        level += 1
    return hop


def gen_diffusion(n: int, steps: int, seed: int, adj=None, sources=None, n_sources: int = 8,
                  period: int = 3, dirty_window: int = 16):
    """Information diffusion along a graph, breadth-first.

    The information reaches BFS level L at step L*period; agents of that level are active
    for ``period`` steps (first WAITING, then GENERATING) and IDLE afterwards (activate at
    most once).  Not-yet-reached agents are ACTING with t_next = remaining hops to
    the wave (hop - level), UNREACHABLE when no path exists.  A new wave with new sources
    starts once the previous one has died out.  Returns phase, t_next, dirty (steps, n)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if adj is None:
        adj = ba_graph(n, 4, seed + 7919)
    P = np.empty((steps, n), np.uint8)
    T = np.empty((steps, n), np.int64)
    D = np.empty((steps, n), np.uint8)
    last_gen = np.full(n, -(10 ** 9), np.int64)
    wave_start = 0
    hop = None
    for s in range(steps):
        if hop is None or s - wave_start >= period * (int(hop[hop != UNREACHABLE].max()) + 2):
            src = sources if (sources is not None and hop is None) else \
                rng.choice(n, size=min(n_sources, n), replace=False)
            hop = bfs_hops(adj, src)
            wave_start = s
        level = (s - wave_start) // period
        k = (s - wave_start) % period
        reach = hop != UNREACHABLE
        ph = np.full(n, PH_IDLE, np.int64)
        tn = np.zeros(n, np.int64)
        ahead = reach & (hop > level)
        ph[ahead] = PH_ACTING
        tn[ahead] = hop[ahead] - level
        ph[~reach] = PH_ACTING
        tn[~reach] = UNREACHABLE
        now_active = reach & (hop == level)
        ph[now_active] = PH_WAITING if k == 0 else PH_GENERATING
        last_gen[now_active] = s
        P[s] = ph
        T[s] = tn
        D[s] = (s - last_gen) < dirty_window
    return P, T, D


def host_pattern(n_bytes: int, seed: int = 0, word_offset: int = 0) -> np.ndarray:
    """Deterministic per-offset byte pattern for the host arena (uint32 words)."""
    w = np.arange(word_offset, word_offset + n_bytes // 4, dtype=np.uint64)
    x = (w * np.uint64(0x9E3779B1) + np.uint64(seed * 0x85EBCA77 + 1)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(15)
    return x.astype(np.uint32)


# ------------------------------------------------------------------------------------
# The five BASELINE.json configs.


def _assemble(name, P, T, D, cls, fp, blocks, budget, theta, kin=None, kin_idx=None, hop_scale=1.0,
              t0=0, meta=None):
    steps, n = P.shape
    rec = np.empty((steps, n, 4), np.uint32)
    ki = np.zeros(n, np.uint32) if kin_idx is None else kin_idx
    for s in range(steps):
        rec[s] = pack_records(T[s], fp, P[s], cls, D[s], ki)
    now = np.arange(t0, t0 + steps, dtype=np.int64)
    return Workload(name, n, now, rec, kin, blocks, int(budget), np.asarray(theta, np.float32),
                    float(hop_scale), PAGE_BYTES, meta or {})


def config_c1(seed: int = 1, theta=(3.0, 3.0, 3.0), steps: int = 8, variant: str = "ind") -> Workload:
    """C1: 16 agents, 8 steps, budget = 4 slots of uniform 1 MiB blocks (BASELINE.json
    configs[0]).  g = 1, action U{1..6}.  Variants: 'ind', 'int' (16 interaction agents),
    'diff' (path graph / star graph)."""
    n = 16
    mib = 1 << 20
    blocks = make_blocks([[KIND_KV]] * n, [[mib]] * n)
    fp = np.full(n, mib, np.uint64)
    if variant == "ind":
        P, T, D = gen_independent(n, steps, seed, g_choices=(1,), fixed_dur=(1, 6))
        cls = np.full(n, CL_IND)
        return _assemble("c1-ind", P, T, D, cls, fp, blocks, 4 * mib, theta)
    if variant == "int":
        P, T, D, K = gen_interaction(n, steps, seed, arena=12.0, r_int=1.0, v_max=1.0,
                                     g_choices=(1,))
        cls = np.full(n, CL_INT)
        return _assemble("c1-int", P, T, D, cls, fp, blocks, 4 * mib, theta, kin=K,
                         kin_idx=np.arange(n, dtype=np.uint32))
    if variant in ("diff", "diff-star"):
        if variant == "diff":
            adj = [[j for j in (i - 1, i + 1) if 0 <= j < n] for i in range(n)]  # path
            src = [0]
        else:
            adj = [list(range(1, n))] + [[0] for _ in range(1, n)]  # star, centre 0
            src = [0]
        P, T, D = gen_diffusion(n, steps, seed, adj=adj, sources=src, period=2)
        cls = np.full(n, CL_DIFF)
        return _assemble("c1-" + variant, P, T, D, cls, fp, blocks, 4 * mib, theta, hop_scale=1.0)
    raise ValueError(variant)


def config_c2(seed: int = 1, steps: int = 64, n: int = 10_000, host_bytes: Optional[int] = None,
              budget_frac: float = 0.25, theta_ind: float = 4.0, lora: int = LORA_7B, kv: int = KV_7B,
              kv_mean: float = 3.0, noise: float = 0.0) -> Workload:
    """C2: AgentSociety-shaped trace, 10k agents, ~5% activated per step, 1 LoRA (rank 16,
    Qwen2.5-7B q/k/v/o) + K ~ 1+Poisson(3) KV pages per agent; budget 25% of the total.
    noise: the S:187 knob (recorded action ends are estimates, gen_independent)."""
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    n_kv = 1 + rng.poisson(kv_mean, size=n)
    blocks = _blocks_vectorized(n, lora, kv, n_kv, 0, host_bytes)
    fp = blocks.footprint
    budget = int(int(fp.sum()) * budget_frac)
    P, T, D = gen_independent(n, steps, seed, active=0.05, noise=noise)
    return _assemble("c2", P, T, D, np.full(n, CL_IND), fp, blocks, budget, (theta_ind, theta_ind, theta_ind),
                     meta=dict(budget_frac=budget_frac))


def config_c3(seed: int = 1, steps: int = 8, n: int = 100_000, host_bytes: Optional[int] = None,
              budget: int = 80 * 10 ** 9, hop_period: int = 3, arena: Optional[float] = None) -> Workload:
    """C3: 100k agents, all three classes (ids [0,n/3) IND, [n/3, 2n/3) INT, rest DIFF),
    5% active, LoRA 0.5B (2,162,688 B) + 1+Poisson(5) KV pages (196,608 B) + 1 HIST (64 KiB);
    80 GB budget; theta = (4, 4, 2*hop_scale), hop_scale = ticks per hop = period."""
    rng = np.random.Generator(np.random.PCG64(seed + 2000))
    a = int(round(n / 3))
    b = int(round(2 * n / 3))
    n_ind, n_int, n_diff = a, b - a, n - b
    n_kv = 1 + rng.poisson(5.0, size=n)
    blocks = _blocks_vectorized(n, LORA_05B, KV_05B, n_kv, HIST, host_bytes)
    fp = blocks.footprint
    Pi, Ti, Di = gen_independent(n_ind, steps, seed, active=0.05)
    if arena is None:
        arena = 2000.0 * np.sqrt(n_int / 33_333.0)
    Pn, Tn, Dn, K = gen_interaction(n_int, steps, seed + 1, active=0.05, arena=arena, r_int=1.0, v_max=1.0)
    Pd, Td, Dd = gen_diffusion(n_diff, steps, seed + 2, period=hop_period)
    P = np.concatenate([Pi, Pn, Pd], axis=1)
    T = np.concatenate([Ti, Tn, Td], axis=1)
    D = np.concatenate([Di, Dn, Dd], axis=1)
    cls = np.concatenate([np.full(n_ind, CL_IND), np.full(n_int, CL_INT), np.full(n_diff, CL_DIFF)])
    kin_idx = np.zeros(n, np.uint32)
    kin_idx[a:b] = np.arange(n_int, dtype=np.uint32)
    hop_scale = float(hop_period)
    return _assemble("c3", P, T, D, cls, fp, blocks, budget, (4.0, 4.0, 2.0 * hop_scale), kin=K,
                     kin_idx=kin_idx, hop_scale=hop_scale)


def config_c4(seed: int = 1, steps: int = 16, n: int = 1_000_000, budget_frac: float = 0.25,
              theta: float = 4.0) -> Workload:
    """C4: 1M independent agents (AgentSociety), C3's footprint distribution with
    logical sizes (no physical transfer), budget 25% of the total, theta = 4."""
    rng = np.random.Generator(np.random.PCG64(seed + 4000))
    n_kv = 1 + rng.poisson(5.0, size=n)
    blocks = _blocks_vectorized(n, LORA_05B, KV_05B, n_kv, HIST, None)
    fp = blocks.footprint
    budget = int(int(fp.sum()) * budget_frac)
    P, T, D = gen_independent(n, steps, seed, active=0.05)
    return _assemble("c4", P, T, D, np.full(n, CL_IND), fp, blocks, budget, (theta, theta, theta),
                     meta=dict(budget_frac=budget_frac))


def config_c5(replica: int, budget_pct: int, seed_base: int = 100, steps: int = 16, n: int = 10_000) -> Workload:
    """C5: one planner instance of the sweep: replica r (seed = base + r) of the C2
    shape with budget = budget_pct% of its total agent memory; plan-only."""
    w = config_c2(seed=seed_base + replica, steps=steps, n=n, budget_frac=budget_pct / 100.0)
    w.name = f"c5-r{replica}-b{budget_pct}"
    return w


def config_by_name(name: str, **kw) -> Workload:
    return {"c1": config_c1, "c2": config_c2, "c3": config_c3, "c4": config_c4}[name](**kw)
