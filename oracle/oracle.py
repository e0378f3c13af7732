"""ctypes marshalling for oracle.cpp (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Holds no planner arithmetic: every number comes from the C++ oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_HDR = os.path.join(_HERE, "oracle.h")
_SO = os.path.join(_HERE, "liboracle.so")

ST_INSUFFICIENT = 1
ST_BAD_RECORD = 2
ST_BAD_KIN = 4
ST_NO_PAGES = 8

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp into liboracle.so (g++, -O2, no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", "-o", tmp, _SRC]
        subprocess.check_call(cmd)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            u64, u32p, f32p, u8p, u64p = C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_float), \
                C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)
            L.oracle_score.argtypes = [u64, u32p, f32p, u64, C.c_int64, C.c_float, f32p, u32p]
            L.oracle_score.restype = None
            L.oracle_score_sampled.argtypes = [u64, u32p, f32p, u64, C.c_int64, C.c_float, u64p, u64, f32p, u32p]
            L.oracle_score_sampled.restype = None
            L.oracle_interaction.argtypes = [u64, u32p, f32p, u64, f32p, u32p]
            L.oracle_interaction.restype = None
            L.oracle_object_min.argtypes = [u64, f32p, u64, u64p, u32p, f32p, u32p]
            L.oracle_object_min.restype = None
            L.oracle_explicit_dist.argtypes = [u64, u32p, f32p, u32p]
            L.oracle_explicit_dist.restype = None
            L.oracle_lru_records.argtypes = [u64, u32p, C.c_int64, u32p, u32p]
            L.oracle_lru_records.restype = None
            L.oracle_bfs_hops.argtypes = [u64, u64p, u32p, u32p, u64, u32p]
            L.oracle_bfs_hops.restype = None
            L.oracle_plan.argtypes = [u64, u32p, f32p, u8p, f32p, u64, u8p, u32p, u64p, u32p, u64p,
                                      u64p, u32p]
            L.oracle_plan.restype = None
            L.oracle_mem_create.argtypes = [u64, u64p, u32p, u64p, u8p, u64, u64, u8p]
            L.oracle_mem_create.restype = C.c_void_p
            L.oracle_mem_destroy.argtypes = [C.c_void_p]
            L.oracle_mem_destroy.restype = None
            L.oracle_mem_apply.argtypes = [C.c_void_p, u32p, u32p, u64, u32p, u64, u64p, u32p, u64p,
                                           u32p, u64p, u32p]
            L.oracle_mem_apply.restype = None
            L.oracle_mem_total_pages.argtypes = [C.c_void_p]
            L.oracle_mem_total_pages.restype = u64
            L.oracle_mem_page_table.argtypes = [C.c_void_p, u32p]
            L.oracle_mem_page_table.restype = None
            L.oracle_mem_pool.argtypes = [C.c_void_p, u64p, u64p, u32p]
            L.oracle_mem_pool.restype = None
            _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def f32_bits(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)


def _rec(rec):
    rec = np.ascontiguousarray(rec, dtype=np.uint32).reshape(-1, 4)
    return rec


def _kin(kin):
    if kin is None or len(kin) == 0:
        return np.zeros((1, 4), dtype=np.float32), 0
    kin = np.ascontiguousarray(kin, dtype=np.float32).reshape(-1, 4)
    return kin, kin.shape[0]


def score(rec, kin, now: int, hop_scale: float = 1.0):
    """Distances of all agents (float32 array) and the status bits."""
    rec = _rec(rec)
    kin, n_kin = _kin(kin)
    n = rec.shape[0]
    d = np.empty(max(n, 1), dtype=np.float32)
    st = np.zeros(1, dtype=np.uint32)
    lib().oracle_score(n, _p(rec, C.c_uint32), _p(kin, C.c_float), n_kin, int(now),
                       float(hop_scale), _p(d, C.c_float), _p(st, C.c_uint32))
    return d[:n], int(st[0])


def score_sampled(rec, kin, now: int, agents, hop_scale: float = 1.0):
    """oracle_score's distances of the given agents only (the Eq. 2 scan over every
    participant for each sampled one)."""
    rec = _rec(rec)
    kin, n_kin = _kin(kin)
    idx = np.ascontiguousarray(agents, dtype=np.uint64)
    d = np.empty(max(len(idx), 1), dtype=np.float32)
    st = np.zeros(1, dtype=np.uint32)
    lib().oracle_score_sampled(rec.shape[0], _p(rec, C.c_uint32), _p(kin, C.c_float), n_kin, int(now),
                               C.c_float(hop_scale), _p(idx, C.c_uint64), len(idx), _p(d, C.c_float),
                               _p(st, C.c_uint32))
    return d[:len(idx)], int(st[0])


def interaction(rec, kin):
    rec = _rec(rec)
    kin, n_kin = _kin(kin)
    dint = np.empty(max(n_kin, 1), dtype=np.float32)
    st = np.zeros(1, dtype=np.uint32)
    lib().oracle_interaction(rec.shape[0], _p(rec, C.c_uint32), _p(kin, C.c_float), n_kin,
                             _p(dint, C.c_float), _p(st, C.c_uint32))
    return dint[:n_kin], int(st[0])


def object_min(agent_dist, ref_ptr, ref_agent):
    """Shared-object distances: float32 [n_objects] and the status bits."""
    ad = np.ascontiguousarray(agent_dist, dtype=np.float32)
    rp = np.ascontiguousarray(ref_ptr, dtype=np.uint64)
    ra = np.ascontiguousarray(ref_agent, dtype=np.uint32)
    n_obj = rp.shape[0] - 1
    out = np.empty(max(n_obj, 1), dtype=np.float32)
    st = np.zeros(1, dtype=np.uint32)
    lib().oracle_object_min(ad.shape[0], _p(ad if ad.size else np.zeros(1, np.float32), C.c_float), n_obj,
                            _p(rp, C.c_uint64), _p(ra if ra.size else np.zeros(1, np.uint32), C.c_uint32),
                            _p(out, C.c_float), _p(st, C.c_uint32))
    return out[:n_obj], int(st[0])


def explicit_dist(rec):
    """Explicit distances of records (reading R19) and the status bits."""
    rec = _rec(rec)
    n = rec.shape[0]
    d = np.empty(max(n, 1), dtype=np.float32)
    st = np.zeros(1, dtype=np.uint32)
    lib().oracle_explicit_dist(n, _p(rec if n else np.zeros((1, 4), np.uint32), C.c_uint32), _p(d, C.c_float),
                               _p(st, C.c_uint32))
    return d[:n], int(st[0])


def lru_records(rec, now: int, last_use):
    """LRU-baseline records (reading R20); last_use (uint32, n) is updated in place."""
    rec = _rec(rec)
    n = rec.shape[0]
    assert last_use.dtype == np.uint32 and last_use.flags.c_contiguous and last_use.shape[0] == n
    out = np.zeros((max(n, 1), 4), dtype=np.uint32)
    lib().oracle_lru_records(n, _p(rec, C.c_uint32), int(now), _p(last_use, C.c_uint32), _p(out, C.c_uint32))
    return out[:n]


def bfs_hops(row_ptr, col, sources):
    """Diffusion hop counts (R9): uint32 BFS levels, 0xFFFFFFFF unreachable."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    cl = np.ascontiguousarray(col, dtype=np.uint32)
    sr = np.ascontiguousarray(sources, dtype=np.uint32)
    n = rp.shape[0] - 1
    out = np.zeros(max(n, 1), dtype=np.uint32)
    lib().oracle_bfs_hops(n, _p(rp, C.c_uint64), _p(cl if cl.size else np.zeros(1, np.uint32), C.c_uint32),
                          _p(sr if sr.size else np.zeros(1, np.uint32), C.c_uint32), sr.shape[0], _p(out, C.c_uint32))
    return out[:n]


def plan(rec, d, resident, theta, budget: int):
    """One planning step.  Returns a dict with resident (u8), prefetch, evict (u32 ids in
    list order), bytes_h2d, cut_bits, cut_rem, kept_bytes, n_eligible, status."""
    rec = _rec(rec)
    n = rec.shape[0]
    d = np.ascontiguousarray(d, dtype=np.float32)
    res_in = np.ascontiguousarray(resident, dtype=np.uint8)
    assert d.shape[0] == n and res_in.shape[0] == n
    th = np.ascontiguousarray(theta, dtype=np.float32)
    assert th.shape[0] == 3
    res_out = np.zeros(max(n, 1), dtype=np.uint8)
    pf = np.zeros(max(n, 1), dtype=np.uint32)
    ev = np.zeros(max(n, 1), dtype=np.uint32)
    npf = np.zeros(1, dtype=np.uint64)
    nev = np.zeros(1, dtype=np.uint64)
    out = np.zeros(5, dtype=np.uint64)
    st = np.zeros(1, dtype=np.uint32)
    if n == 0:
        d = np.zeros(1, dtype=np.float32)
        res_in = np.zeros(1, dtype=np.uint8)
        rec = np.zeros((1, 4), dtype=np.uint32)
    lib().oracle_plan(n, _p(rec, C.c_uint32), _p(d, C.c_float), _p(res_in, C.c_uint8),
                      _p(th, C.c_float), int(budget), _p(res_out, C.c_uint8), _p(pf, C.c_uint32),
                      _p(npf, C.c_uint64), _p(ev, C.c_uint32), _p(nev, C.c_uint64),
                      _p(out, C.c_uint64), _p(st, C.c_uint32))
    return dict(resident=res_out[:n].copy(), prefetch=pf[:int(npf[0])].copy(),
                evict=ev[:int(nev[0])].copy(), bytes_h2d=int(out[0]), cut_bits=int(out[1]),
                cut_rem=int(out[2]), kept_bytes=int(out[3]), n_eligible=int(out[4]),
                status=int(st[0]))


class OracleMem:
    """Paged device-arena bookkeeping (FIFO free-page pool) of oracle.cpp."""

    def __init__(self, blk_ptr, blk_size, blk_host_off, blk_kind, page_bytes: int, n_pages: int,
                 resident_init=None):
        self.blk_ptr = np.ascontiguousarray(blk_ptr, dtype=np.uint64)
        self.blk_size = np.ascontiguousarray(blk_size, dtype=np.uint32)
        self.blk_host_off = np.ascontiguousarray(blk_host_off, dtype=np.uint64)
        self.blk_kind = np.ascontiguousarray(blk_kind, dtype=np.uint8)
        self.n_agents = self.blk_ptr.shape[0] - 1
        self.page_bytes = int(page_bytes)
        self.n_pages = int(n_pages)
        ri = None
        if resident_init is not None:
            ri = np.ascontiguousarray(resident_init, dtype=np.uint8)
        nb = max(self.blk_size.shape[0], 1)
        bs = self.blk_size if self.blk_size.shape[0] else np.zeros(nb, np.uint32)
        bo = self.blk_host_off if self.blk_host_off.shape[0] else np.zeros(nb, np.uint64)
        bk = self.blk_kind if self.blk_kind.shape[0] else np.zeros(nb, np.uint8)
        self._keep = (bs, bo, bk, ri)
        self.h = lib().oracle_mem_create(
            self.n_agents, _p(self.blk_ptr, C.c_uint64), _p(bs, C.c_uint32), _p(bo, C.c_uint64),
            _p(bk, C.c_uint8), self.page_bytes, self.n_pages,
            _p(ri, C.c_uint8) if ri is not None else None)
        self.total_pages = int(lib().oracle_mem_total_pages(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().oracle_mem_destroy(h)
            self.h = None

    def apply(self, rec, prefetch, evict):
        rec = _rec(rec)
        pf = np.ascontiguousarray(prefetch, dtype=np.uint32)
        ev = np.ascontiguousarray(evict, dtype=np.uint32)
        cap = max(self.total_pages, 1)
        d2h_host = np.zeros(cap, np.uint64)
        d2h_page = np.zeros(cap, np.uint32)
        h2d_host = np.zeros(cap, np.uint64)
        h2d_page = np.zeros(cap, np.uint32)
        out = np.zeros(4, np.uint64)
        st = np.zeros(1, np.uint32)
        pf_ = pf if pf.shape[0] else np.zeros(1, np.uint32)
        ev_ = ev if ev.shape[0] else np.zeros(1, np.uint32)
        lib().oracle_mem_apply(self.h, _p(rec, C.c_uint32), _p(pf_, C.c_uint32), pf.shape[0],
                               _p(ev_, C.c_uint32), ev.shape[0], _p(d2h_host, C.c_uint64),
                               _p(d2h_page, C.c_uint32), _p(h2d_host, C.c_uint64),
                               _p(h2d_page, C.c_uint32), _p(out, C.c_uint64), _p(st, C.c_uint32))
        nd, nh = int(out[2]), int(out[3])
        return dict(bytes_d2h=int(out[0]), bytes_h2d=int(out[1]),
                    d2h_host=d2h_host[:nd].copy(), d2h_page=d2h_page[:nd].copy(),
                    h2d_host=h2d_host[:nh].copy(), h2d_page=h2d_page[:nh].copy(),
                    status=int(st[0]))

    def page_table(self):
        pt = np.zeros(max(self.total_pages, 1), np.uint32)
        lib().oracle_mem_page_table(self.h, _p(pt, C.c_uint32))
        return pt[:self.total_pages]

    def pool(self):
        head = np.zeros(1, np.uint64)
        tail = np.zeros(1, np.uint64)
        ring = np.zeros(max(self.n_pages, 1), np.uint32)
        lib().oracle_mem_pool(self.h, _p(head, C.c_uint64), _p(tail, C.c_uint64), _p(ring, C.c_uint32))
        return int(head[0]), int(tail[0]), ring[:self.n_pages]
