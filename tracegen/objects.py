"""Shared memory objects over an agent population: a system-prompt
prefix shared by every agent, persona LoRA adapters each shared by a group of agents, and
every agent's private KV pages.  Only the reference structure (CSR object -> referencing
agents), the sizes and the per-step dirty flags; none of the planner's arithmetic."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .traces import KIND_KV, KIND_LORA, KV_7B, LORA_7B, PAGE_BYTES, Blocks


@dataclass
class Objects:
    ref_ptr: np.ndarray    # (n_obj + 1,) uint64 CSR offsets
    ref_agent: np.ndarray  # (refs,) uint32 referencing agents
    obj_bytes: np.ndarray  # (n_obj,) uint32
    obj_kind: np.ndarray   # (n_obj,) uint8 (KIND_LORA adapters are never written back)
    private_of: np.ndarray  # (n_agents,) object index of each agent's private pages
    blocks: Blocks         # one block per object (the object planner's block table)

    @property
    def n(self) -> int:
        return len(self.obj_bytes)

    def flags(self, agent_rec: np.ndarray) -> np.ndarray:
        """Per-object flags word for one step: an agent's private pages carry its dirty bit;
        the shared prompt prefix and the adapters are read-only (flags 0, class 0, ACTING)."""
        f = np.zeros(self.n, dtype=np.uint32)
        f[self.private_of] = agent_rec[:, 2] & np.uint32(1 << 4)
        return f


def gen_objects(n_agents: int, seed: int = 1, personas: Optional[int] = None, prompt_pages: int = 64,
                kv: int = KV_7B, lora: int = LORA_7B, kv_mean: float = 3.0,
                host_bytes: Optional[int] = None) -> Objects:
    """Object 0: system prompt (prompt_pages KV pages), referenced by every agent.
    Objects 1..P: persona adapters (rank-16 LoRA), agent a uses persona ~ U{0..P-1}.
    Objects P+1..P+n: agent a's private KV pages, 1 + Poisson(kv_mean) pages."""
    rng = np.random.Generator(np.random.PCG64(seed + 7000))
    P = personas if personas is not None else max(1, n_agents // 100)
    persona = rng.integers(0, P, n_agents)
    n_obj = 1 + P + n_agents
    agents = np.arange(n_agents, dtype=np.uint32)
    # CSR: prompt -> all agents; persona p -> its agents (ascending id); private -> its agent
    order = np.argsort(persona, kind="stable")
    per_cnt = np.bincount(persona, minlength=P)
    cnt = np.concatenate([[n_agents], per_cnt, np.ones(n_agents, np.int64)])
    ref_ptr = np.zeros(n_obj + 1, dtype=np.uint64)
    ref_ptr[1:] = np.cumsum(cnt)
    ref_agent = np.concatenate([agents, agents[order], agents]).astype(np.uint32)
    n_kv = 1 + rng.poisson(kv_mean, size=n_agents)
    obj_bytes = np.concatenate([[prompt_pages * kv], np.full(P, lora), n_kv * kv]).astype(np.uint64)
    assert np.all(obj_bytes % PAGE_BYTES == 0) and np.all(obj_bytes < 2**32)
    obj_kind = np.concatenate([[KIND_KV], np.full(P, KIND_LORA), np.full(n_agents, KIND_KV)]).astype(np.uint8)
    off = np.zeros(n_obj, dtype=np.uint64)
    off[1:] = np.cumsum(obj_bytes)[:-1]
    total = int(obj_bytes.sum())
    if host_bytes is not None and total > host_bytes:  # aliased modulo the pinned arena (bytes moved are real)
        span = host_bytes - int(obj_bytes.max())
        off = (off % np.uint64(span)) // np.uint64(PAGE_BYTES) * np.uint64(PAGE_BYTES)
    blocks = Blocks(np.arange(n_obj + 1, dtype=np.uint64), obj_bytes.astype(np.uint32), off, obj_kind,
                    host_bytes if host_bytes is not None else total)
    return Objects(ref_ptr, ref_agent, obj_bytes.astype(np.uint32), obj_kind,
                   (1 + P + np.arange(n_agents)).astype(np.int64), blocks)


def object_records(d_bits: np.ndarray, obj: Objects, flags: np.ndarray) -> np.ndarray:
    """Explicit-distance records (R19): word 0 = the given distance bits."""
    rec = np.zeros((obj.n, 4), dtype=np.uint32)
    rec[:, 0] = d_bits
    rec[:, 1] = obj.obj_bytes
    rec[:, 2] = flags
    return rec
