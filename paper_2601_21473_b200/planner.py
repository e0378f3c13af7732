"""Thin Python binding of the C ABI.  PyTorch provides device / pinned memory and streams
only; every step of the planner runs in libscalesim.so's kernels.  Names follow
include/scalesim.h (score / plan / transfer / step / sync)."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib as L


def _dev_bytes(arr: np.ndarray, device) -> torch.Tensor:
    a = np.ascontiguousarray(arr)
    t = torch.from_numpy(a.view(np.uint8).reshape(-1)) if a.nbytes else torch.zeros(16, dtype=torch.uint8)
    return t.to(device)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Planner:
    """One planner context (one rank's shard).

    blk_ptr/blk_size/blk_host_off/blk_kind: numpy CSR block table of the local agents.
    host_arena: pinned uint8 torch tensor (or None: allocated, size host_bytes).
    dev_bytes: HBM arena size (default: ceil(budget / page) pages).
    """

    def __init__(self, n_agents: int, blk_ptr, blk_size, blk_host_off, blk_kind, budget: int, theta,
                 hop_scale: float = 1.0, n_kin: int = 0, page_bytes: int = 65536, transfer: bool = True,
                 host_arena: Optional[torch.Tensor] = None, host_bytes: Optional[int] = None,
                 dev_bytes: Optional[int] = None, resident_init=None, device: int = 0,
                 shard: Optional[tuple] = None, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 stream: Optional[torch.cuda.Stream] = None, copy_stream: Optional[torch.cuda.Stream] = None,
                 multi_kernel: bool = False, keep_dist: bool = True, explicit_dist: bool = False,
                 exclusive: bool = False, loopback: bool = False, tp_sliced: bool = False, threads: bool = False):
        self.lib = L.lib()
        self._staged_refs = {}  # host arrays of staged steps (scalesim_stage_host)
        self._pending = []  # host arrays of submitted, uncollected steps (scalesim_submit_updates)
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        lo, hi = shard if shard is not None else (0, n_agents)
        self.n_agents, self.lo, self.hi = int(n_agents), int(lo), int(hi)
        self.n_local = self.hi - self.lo
        self.n_kin = int(n_kin)
        self.page_bytes = int(page_bytes)
        self.transfer_enabled = bool(transfer)
        self.stream = stream or torch.cuda.Stream(self.device)
        self.copy_stream = copy_stream or torch.cuda.Stream(self.device)
        dev = self.device
        # inputs
        self.rec = torch.zeros(max(self.n_local, 1) * 16, dtype=torch.uint8, device=dev)
        self.kin = torch.zeros(max(self.n_kin, 1) * 16, dtype=torch.uint8, device=dev)
        blk_ptr = np.ascontiguousarray(blk_ptr, dtype=np.uint64)
        blk_size = np.ascontiguousarray(blk_size, dtype=np.uint32)
        self.n_blocks = int(blk_ptr[-1]) if len(blk_ptr) else 0
        self.blk_ptr = _dev_bytes(blk_ptr, dev)
        self.blk_size = _dev_bytes(blk_size, dev)
        self.blk_host_off = _dev_bytes(np.ascontiguousarray(blk_host_off, dtype=np.uint64), dev)
        self.blk_kind = _dev_bytes(np.ascontiguousarray(blk_kind, dtype=np.uint8), dev)
        self.n_block_pages = int((blk_size.astype(np.uint64) // np.uint64(page_bytes)).sum()) if transfer else 0
        self.blk_size_np = blk_size
        self.budget = int(budget)
        # arenas
        self.host_arena = None
        self.dev_arena = None
        if transfer:
            if host_arena is None:
                hb = int(host_bytes) if host_bytes is not None else int(np.asarray(blk_host_off, np.uint64).max(
                    initial=0) + page_bytes + (int(blk_size.max()) if len(blk_size) else 0))
                host_arena = torch.zeros(hb, dtype=torch.uint8, pin_memory=True)
            self.host_arena = host_arena
            if dev_bytes is None:  # (TP-sliced: a slot holds this rank's 1/world of a page)
                dev_bytes = (self.budget + page_bytes - 1) // page_bytes * (page_bytes // (world if tp_sliced else 1))
            self.dev_arena = torch.empty(max(int(dev_bytes), page_bytes), dtype=torch.uint8, device=dev)
        self.res_init = None
        if resident_init is not None:
            ri = np.ascontiguousarray(resident_init).astype(bool)
            words = np.packbits(ri, bitorder="little")
            pad = (-len(words)) % 4
            words = np.concatenate([words, np.zeros(pad, np.uint8)])
            self.res_init = _dev_bytes(words, dev)
        self._nccl_id = None
        if world > 1 and not loopback:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
        cfg = L.Config()
        cfg.abi_version = L.ABI_VERSION
        cfg.flags = (0 if transfer else L.F_NO_TRANSFER) | (L.F_MULTI_KERNEL if multi_kernel else 0) | \
            (L.F_KEEP_DIST if keep_dist else 0) | (L.F_EXPLICIT_DIST if explicit_dist else 0) | \
            (L.F_EXCLUSIVE if exclusive else 0) | (L.F_LOOPBACK if loopback else 0) | \
            (L.F_TP_SLICED if tp_sliced else 0) | (L.F_THREADS if threads else 0)
        self.tp_sliced = bool(tp_sliced)
        self.slot_bytes = self.page_bytes // (world if tp_sliced else 1)
        cfg.n_agents = self.n_agents
        cfg.shard_begin = self.lo
        cfg.shard_end = self.hi
        cfg.n_kin = self.n_kin
        cfg.budget_bytes = self.budget
        th = np.asarray(theta, dtype=np.float32)
        cfg.theta[0], cfg.theta[1], cfg.theta[2] = float(th[0]), float(th[1]), float(th[2])
        cfg.hop_scale = float(hop_scale)
        cfg.page_bytes = self.page_bytes
        cfg.device = int(device)
        cfg.rank = int(rank)
        cfg.world = int(world)
        cfg.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None
        cfg.stream = self.stream.cuda_stream
        cfg.copy_stream = self.copy_stream.cuda_stream
        self.cfg = cfg
        tab = L.Tables()
        tab.agent_rec = _ptr(self.rec)
        tab.agent_kin = _ptr(self.kin)
        tab.blk_ptr = _ptr(self.blk_ptr)
        tab.blk_size = _ptr(self.blk_size)
        tab.blk_host_off = _ptr(self.blk_host_off)
        tab.blk_kind = _ptr(self.blk_kind)
        tab.n_blocks = self.n_blocks
        tab.n_block_pages = self.n_block_pages
        tab.host_arena = _ptr(self.host_arena)
        tab.host_bytes = 0 if self.host_arena is None else self.host_arena.numel()
        tab.dev_arena = _ptr(self.dev_arena)
        tab.dev_bytes = 0 if self.dev_arena is None else self.dev_arena.numel()
        tab.resident_init = _ptr(self.res_init)
        ws = int(self.lib.scalesim_workspace_bytes(C.byref(cfg), C.byref(tab)))
        if ws == 0:
            raise L.ScaleSimError(L.E_INVALID, "scalesim_workspace_bytes")
        self.workspace = torch.empty(ws + 256, dtype=torch.uint8, device=dev)
        base = self.workspace.data_ptr()
        tab.workspace = (base + 255) // 256 * 256
        tab.workspace_bytes = ws
        self.tab = tab
        self.ctx = C.c_void_p()
        torch.cuda.synchronize(self.device)
        L.check(self.lib.scalesim_init(C.byref(cfg), C.byref(tab), C.byref(self.ctx)), "scalesim_init")
        self.view = L.PlanView()

    # ---- inputs ------------------------------------------------------------------
    def set_records(self, rec, kin=None):
        """Copy this step's agent records (n_local, 4) uint32 and kinematics to the device
        buffers the context reads (on the planner stream)."""
        with torch.cuda.stream(self.stream):
            r = np.ascontiguousarray(rec, dtype=np.uint32)
            assert r.size == 4 * self.n_local
            if self.n_local:
                self.rec[:r.nbytes].copy_(torch.from_numpy(r.view(np.uint8).reshape(-1)), non_blocking=False)
            if kin is not None and self.n_kin:
                k = np.ascontiguousarray(kin, dtype=np.float32)
                self.kin[:k.nbytes].copy_(torch.from_numpy(k.view(np.uint8).reshape(-1)), non_blocking=False)

    def set_inputs_ptr(self, rec_ptr: int, kin_ptr: Optional[int] = None):
        L.check(self.lib.scalesim_set_inputs(self.ctx, rec_ptr, kin_ptr or _ptr(self.kin)), "scalesim_set_inputs")

    # ---- the four calls ------------------------------------------------------------
    def score(self, now: int, dist_out: Optional[torch.Tensor] = None):
        L.check(self.lib.scalesim_score(self.ctx, int(now), _ptr(dist_out)), "scalesim_score")

    def plan(self):
        L.check(self.lib.scalesim_plan(self.ctx, C.byref(self.view)), "scalesim_plan")
        return self.view

    def transfer(self):
        L.check(self.lib.scalesim_transfer(self.ctx, C.byref(self.view)), "scalesim_transfer")

    def step(self, now: int):
        L.check(self.lib.scalesim_step(self.ctx, int(now), C.byref(self.view)), "scalesim_step")
        return self.view

    def step_host(self, now: int, rec_host: np.ndarray, kin_host: Optional[np.ndarray] = None,
                  pf_out: Optional[np.ndarray] = None, ev_out: Optional[np.ndarray] = None):
        """End-to-end step from host buffers (host->device copy, step, header + lists back)."""
        h = L.PlanHost()
        rp = rec_host.ctypes.data
        kp = kin_host.ctypes.data if kin_host is not None else None
        st = self.lib.scalesim_step_host(self.ctx, int(now), rp, kp, C.byref(h),
                                         None if pf_out is None else pf_out.ctypes.data,
                                         None if ev_out is None else ev_out.ctypes.data)
        self._staged_refs.pop(rp, None)
        L.check(st, "scalesim_step_host", allow=(L.OK, L.E_INSUFFICIENT))
        return h.as_dict()

    def stage_host(self, rec_host: np.ndarray, kin_host: Optional[np.ndarray] = None):
        """Start the host->device copy of a later step's inputs (scalesim_stage_host); the
        step_host call with the same arrays plans from the staged copy.  The arrays are kept
        alive here until that call."""
        kp = kin_host.ctypes.data if kin_host is not None else None
        L.check(self.lib.scalesim_stage_host(self.ctx, rec_host.ctypes.data, kp), "scalesim_stage_host")
        self._staged_refs[rec_host.ctypes.data] = (rec_host, kin_host)

    def stage_updates(self, ids: np.ndarray, recs: np.ndarray):
        """Start the host->device copy of a later step's changed records (scalesim_stage_updates):
        ids (n,) uint32 global agent ids, recs (n, 4) uint32, both C-contiguous (pinned for an
        asynchronous copy).  Kept alive here until the matching step_updates."""
        assert ids.dtype == np.uint32 and recs.dtype == np.uint32 and recs.shape == (len(ids), 4)
        L.check(self.lib.scalesim_stage_updates(self.ctx, ids.ctypes.data, recs.ctypes.data, len(ids)),
                "scalesim_stage_updates")
        self._staged_refs[ids.ctypes.data] = (ids, recs)

    def step_updates(self, now: int, ids: np.ndarray, recs: np.ndarray, pf_out: Optional[np.ndarray] = None,
                     ev_out: Optional[np.ndarray] = None):
        """Incremental end-to-end step (scalesim_step_updates): the changed records scattered into
        the context's record buffer, the step, header + lists back."""
        assert ids.dtype == np.uint32 and recs.dtype == np.uint32 and recs.shape == (len(ids), 4)
        h = L.PlanHost()
        st = self.lib.scalesim_step_updates(self.ctx, int(now), ids.ctypes.data, recs.ctypes.data, len(ids),
                                            C.byref(h), None if pf_out is None else pf_out.ctypes.data,
                                            None if ev_out is None else ev_out.ctypes.data)
        self._staged_refs.pop(ids.ctypes.data, None)
        L.check(st, "scalesim_step_updates", allow=(L.OK, L.E_INSUFFICIENT))
        return h.as_dict()

    def submit_updates(self, now: int, ids: np.ndarray, recs: np.ndarray):
        """Enqueue an incremental step and return at once (scalesim_submit_updates); its
        header and lists come back from collect(), oldest first."""
        assert ids.dtype == np.uint32 and recs.dtype == np.uint32 and recs.shape == (len(ids), 4)
        L.check(self.lib.scalesim_submit_updates(self.ctx, int(now), ids.ctypes.data, recs.ctypes.data, len(ids)),
                "scalesim_submit_updates")
        self._pending.append((ids, recs))

    def collect(self, pf_out: Optional[np.ndarray] = None, ev_out: Optional[np.ndarray] = None):
        """Header (dict) and lists of the oldest submitted step (scalesim_collect)."""
        h = L.PlanHost()
        st = self.lib.scalesim_collect(self.ctx, C.byref(h), None if pf_out is None else pf_out.ctypes.data,
                                       None if ev_out is None else ev_out.ctypes.data)
        if self._pending:
            self._pending.pop(0)
        L.check(st, "scalesim_collect", allow=(L.OK, L.E_INSUFFICIENT))
        return h.as_dict()

    def join(self):
        L.check(self.lib.scalesim_join(self.ctx), "scalesim_join")

    def sync(self):
        h = L.PlanHost()
        st = self.lib.scalesim_sync(self.ctx, C.byref(h))
        L.check(st, "scalesim_sync", allow=(L.OK, L.E_INSUFFICIENT, L.E_BAD_INPUT))
        d = h.as_dict()
        d["rc"] = st
        return d

    def stamps(self, reset: bool = False) -> np.ndarray:
        """The fused kernel's %globaltimer stamps (ns), see scalesim_profile_stamps."""
        ptr = int(self.lib.scalesim_profile_stamps(self.ctx))
        v = self._read(ptr, 512).view(np.uint64).copy()
        if reset:
            off = ptr - self.workspace.data_ptr()
            init = np.zeros(64, np.uint64)
            init[0] = np.iinfo(np.uint64).max
            self.workspace[off:off + 512].copy_(torch.from_numpy(init.view(np.uint8)))
            torch.cuda.synchronize(self.device)
        return v

    def list_paths(self):
        """(fast, slow): fused launches so far whose lists were placed from the published
        counts (no second grid barrier) / by the staged per-bucket sort."""
        v = self.stamps()
        return int(v[48]), int(v[49])

    @property
    def fused(self) -> bool:
        return int(self.lib.scalesim_fused(self.ctx)) >= 1

    @property
    def big(self) -> bool:
        """The streaming single-kernel plan of large integer-distance contexts."""
        return int(self.lib.scalesim_fused(self.ctx)) == 2

    def launch_count(self) -> int:
        return int(self.lib.scalesim_launch_count(self.ctx))

    # ---- readbacks (tests / tools) --------------------------------------------------
    def _read(self, ptr: int, nbytes: int) -> np.ndarray:
        """Copy nbytes at a view pointer (always inside the workspace) to the host."""
        off = int(ptr) - self.workspace.data_ptr()
        assert 0 <= off and off + nbytes <= self.workspace.numel()
        torch.cuda.synchronize(self.device)
        return self.workspace[off:off + nbytes].cpu().numpy()

    def lists(self, hdr=None):
        hdr = hdr or self.sync()
        pf = self._read(self.view.prefetch_ids, 4 * hdr["n_prefetch"]).view(np.uint32)
        ev = self._read(self.view.evict_ids, 4 * hdr["n_evict"]).view(np.uint32)
        return pf, ev

    def resident(self) -> np.ndarray:
        nw = (self.n_local + 31) // 32
        words = self._read(self.view.resident_bitmap, 4 * nw)
        return np.unpackbits(words, bitorder="little")[:self.n_local].astype(np.uint8)

    def distances(self) -> np.ndarray:
        return self._read(self.view.dist, 4 * self.n_local).view(np.float32)

    def dist_tensor(self) -> torch.Tensor:
        """Device view (float32, n_local) of the distances of the last plan (keep_dist)."""
        off = int(self.view.dist) - self.workspace.data_ptr()
        return self.workspace[off: off + 4 * self.n_local].view(torch.float32)

    def page_table(self) -> np.ndarray:
        return self._read(self.view.page_table, 4 * self.n_block_pages).view(np.uint32)

    def world_lists(self):
        """TP-sliced rank: the world's merged prefetch / evict lists and header fields after the
        last step (scalesim_world_view)."""
        wv = L.WorldView()
        L.check(self.lib.scalesim_world_view(self.ctx, C.byref(wv)), "scalesim_world_view")
        h = self._read(wv.header, 8 * 16).view(np.uint64)
        hdr = dict(n_prefetch=int(h[0]), n_evict=int(h[1]), bytes_d2h=int(h[3]), n_d2h=int(h[7]), n_h2d=int(h[8]),
                   status=int(h[6]))
        pf = self._read(wv.prefetch_ids, 4 * hdr["n_prefetch"]).view(np.uint32)
        ev = self._read(wv.evict_ids, 4 * hdr["n_evict"]).view(np.uint32)
        return pf, ev, hdr

    def descriptors(self, hdr=None):
        hdr = hdr or self.sync()
        d2h = self._read(self.view.d2h_desc, 16 * hdr["n_d2h"]).view(np.uint64).reshape(-1, 2)
        h2d = self._read(self.view.h2d_desc, 16 * hdr["n_h2d"]).view(np.uint64).reshape(-1, 2)
        return d2h, h2d

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.scalesim_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



def object_min(agent_dist: torch.Tensor, ref_ptr: torch.Tensor, ref_agent: torch.Tensor, obj_bytes: torch.Tensor,
               rec_out: torch.Tensor, obj_flags: Optional[torch.Tensor] = None, dist_out: Optional[torch.Tensor] = None,
               status: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None):
    """scalesim_object_min: shared-object distances (min over referencing agents)
    written as explicit-distance records into rec_out (uint8 device tensor, 16 B per object).
    All tensors on the same CUDA device; ref_ptr int64/uint64 [n_objects + 1], ref_agent,
    obj_bytes, obj_flags 32-bit."""
    lib = L.lib()
    n_obj = ref_ptr.numel() - 1
    st = stream if stream is not None else torch.cuda.current_stream(agent_dist.device)
    L.check(lib.scalesim_object_min(_ptr(agent_dist), agent_dist.numel(), _ptr(ref_ptr), _ptr(ref_agent), n_obj,
                                    _ptr(obj_bytes), _ptr(obj_flags), _ptr(rec_out), _ptr(dist_out), _ptr(status),
                                    st.cuda_stream), "scalesim_object_min")


def bfs_hops(row_ptr: torch.Tensor, col: torch.Tensor, sources: torch.Tensor,
             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """scalesim_bfs_hops: BFS level of every vertex from the sources (uint32 as int32 tensor,
    -1 = unreachable).  row_ptr int64 [n + 1], col / sources 32-bit, all on one CUDA device."""
    lib = L.lib()
    n = row_ptr.numel() - 1
    dev = row_ptr.device
    hops = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    nb = int(lib.scalesim_bfs_scratch_bytes(n))
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    L.check(lib.scalesim_bfs_hops(_ptr(row_ptr), _ptr(col), n, _ptr(sources), sources.numel(), _ptr(hops),
                                  _ptr(scratch), nb, st.cuda_stream), "scalesim_bfs_hops")
    return hops[:n]


def step_batch(planners, now: int):
    """One step of several independent planners (replicas / sweep points) sharing one stream:
    scalesim_step_batch plans them in as few launches as possible."""
    if not planners:
        return
    lib = planners[0].lib
    arr = (C.c_void_p * len(planners))(*[pl.ctx.value for pl in planners])
    L.check(lib.scalesim_step_batch(arr, len(planners), int(now)), "scalesim_step_batch")
    for pl in planners:
        L.check(lib.scalesim_view(pl.ctx, C.byref(pl.view)), "scalesim_view")


def step_group(ranks, now: int):
    """One step of a world whose ranks (Planner contexts created with loopback=True, rank r
    = ranks[r]) all live on this device: scalesim_step_group plans them in one launch, the
    global cut exchanged through device memory (include/scalesim.h)."""
    lib = ranks[0].lib
    arr = (C.c_void_p * len(ranks))(*[pl.ctx.value for pl in ranks])
    L.check(lib.scalesim_step_group(arr, len(ranks), int(now)), "scalesim_step_group")
    for pl in ranks:
        L.check(lib.scalesim_view(pl.ctx, C.byref(pl.view)), "scalesim_view")


# NEXT #2: the preemptive load scheduler (scalesim_sched_run, include/scalesim.h)
LOAD_EVENT = np.dtype([("slot", "<u4"), ("kind", "<u4"), ("agent", "<u4"), ("priority", "<f4"),
                       ("host_off", "<u8"), ("dev_off", "<u8"), ("bytes", "<u8")])
LOAD_TASK = np.dtype([("agent", "<u4"), ("chunks", "<u4"), ("done", "<u4"), ("state", "<u4"), ("priority", "<f4"),
                      ("preemptions", "<u4"), ("finish_slot", "<u4"), ("pad", "<u4")])


def sched_run(events: np.ndarray, n_agents: int, threshold: float, chunk_bytes: int, host_arena: torch.Tensor,
              dev_arena: torch.Tensor, max_slots: int, stream: Optional[torch.cuda.Stream] = None, sync: bool = True):
    """Run a load schedule on the device.  events: numpy array of LOAD_EVENT sorted by slot.
    Returns (trace (slots, 2) uint32, tasks LOAD_TASK array, n_slots) after a sync, or the
    device tensors when sync is False."""
    lib = L.lib()
    dev = dev_arena.device
    ev = torch.from_numpy(np.ascontiguousarray(events, dtype=LOAD_EVENT).view(np.uint8)).to(dev)
    n_ev = len(events)
    trace = torch.zeros(max(max_slots, 1) * 2, dtype=torch.int32, device=dev)
    tasks = torch.zeros(max(n_ev, 1) * LOAD_TASK.itemsize, dtype=torch.uint8, device=dev)
    counts = torch.zeros(2, dtype=torch.int32, device=dev)
    nb = int(lib.scalesim_sched_scratch_bytes(n_ev, n_agents))
    scratch = torch.empty(nb + 256, dtype=torch.uint8, device=dev)
    sp = (scratch.data_ptr() + 255) // 256 * 256
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    L.check(lib.scalesim_sched_run(_ptr(ev) if n_ev else None, n_ev, n_agents, float(threshold), int(chunk_bytes),
                                   _ptr(host_arena), _ptr(dev_arena), int(max_slots), _ptr(trace), _ptr(tasks),
                                   _ptr(counts), sp, nb, st.cuda_stream), "scalesim_sched_run")
    if not sync:
        return trace, tasks, counts, (ev, scratch)
    torch.cuda.synchronize(dev)
    c = counts.cpu().numpy().view(np.uint32)
    tr = trace.cpu().numpy().view(np.uint32).reshape(-1, 2)[:c[0]]
    tk = tasks.cpu().numpy()[:c[1] * LOAD_TASK.itemsize].view(LOAD_TASK)
    return tr, tk, int(c[0])
