"""ctypes declarations of include/scalesim.h (argument marshalling only).

Loading fails loudly when libscalesim.so is missing: there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("SCALESIM_SO") or os.path.join(HERE, "libscalesim.so")  # override: tools/ A/B runs only

ABI_VERSION = 1
F_NO_TRANSFER = 1
F_KEEP_DIST = 2
F_MULTI_KERNEL = 4
F_EXPLICIT_DIST = 8
F_EXCLUSIVE = 16
F_LOOPBACK = 32
F_TP_SLICED = 64
F_THREADS = 128

ST_INSUFFICIENT = 1
ST_BAD_RECORD = 2
ST_BAD_KIN = 4
ST_NO_PAGES = 8

OK, E_INVALID, E_INSUFFICIENT, E_NOT_RESTORABLE, E_ORDER, E_CUDA, E_NCCL, E_INVARIANT, E_BAD_INPUT = range(9)

H_N_PREFETCH, H_N_EVICT, H_BYTES_H2D, H_BYTES_D2H, H_CUT_BITS, H_CUT_REM, H_STATUS, H_N_D2H, H_N_H2D, \
    H_KEPT_BYTES, H_N_ELIGIBLE, H_POOL_HEAD, H_POOL_TAIL, H_SEQ = range(14)
H_FIELDS = 16
HEADER_NAMES = ["n_prefetch", "n_evict", "bytes_h2d", "bytes_d2h", "cut_bits", "cut_rem", "status",
                "n_d2h", "n_h2d", "kept_bytes", "n_eligible", "pool_head", "pool_tail", "seq"]

# Every symbol include/scalesim.h declares (checked by tests/test_abi.py).
EXPORTS = ["scalesim_workspace_bytes", "scalesim_init", "scalesim_score", "scalesim_plan",
           "scalesim_transfer", "scalesim_view", "scalesim_step", "scalesim_step_batch", "scalesim_step_group", "scalesim_world_view", "scalesim_step_host", "scalesim_stage_host", "scalesim_stage_updates", "scalesim_step_updates", "scalesim_submit_updates", "scalesim_collect", "scalesim_set_inputs",
           "scalesim_sync", "scalesim_join", "scalesim_nccl_unique_id", "scalesim_fused", "scalesim_profile_stamps", "scalesim_object_min", "scalesim_lru_records", "scalesim_bfs_scratch_bytes", "scalesim_bfs_hops", "scalesim_sched_scratch_bytes", "scalesim_sched_run", "scalesim_launch_count", "scalesim_destroy",
           "scalesim_strerror"]


class Config(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("flags", C.c_uint32),
        ("n_agents", C.c_uint64), ("shard_begin", C.c_uint64), ("shard_end", C.c_uint64),
        ("n_kin", C.c_uint64), ("budget_bytes", C.c_uint64),
        ("theta", C.c_float * 3), ("hop_scale", C.c_float),
        ("page_bytes", C.c_uint64),
        ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("copy_stream", C.c_void_p),
    ]


class Tables(C.Structure):
    _fields_ = [
        ("agent_rec", C.c_void_p), ("agent_kin", C.c_void_p),
        ("blk_ptr", C.c_void_p), ("blk_size", C.c_void_p), ("blk_host_off", C.c_void_p),
        ("blk_kind", C.c_void_p), ("n_blocks", C.c_uint64), ("n_block_pages", C.c_uint64),
        ("host_arena", C.c_void_p), ("host_bytes", C.c_uint64),
        ("dev_arena", C.c_void_p), ("dev_bytes", C.c_uint64),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
        ("resident_init", C.c_void_p),
    ]


class WorldView(C.Structure):
    _fields_ = [("prefetch_ids", C.c_void_p), ("evict_ids", C.c_void_p), ("header", C.c_void_p)]


class PlanView(C.Structure):
    _fields_ = [
        ("prefetch_ids", C.c_void_p), ("evict_ids", C.c_void_p), ("resident_bitmap", C.c_void_p),
        ("dist", C.c_void_p), ("page_table", C.c_void_p), ("d2h_desc", C.c_void_p),
        ("h2d_desc", C.c_void_p), ("header", C.c_void_p), ("done_event", C.c_void_p),
    ]


class PlanHost(C.Structure):
    _fields_ = [("f", C.c_uint64 * H_FIELDS)]

    def as_dict(self):
        return {name: int(self.f[k]) for k, name in enumerate(HEADER_NAMES)}


class ScaleSimError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {strerror(status)} ({status})")


_lib = None


def lib():
    """Load libscalesim.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} is missing: run `python -m paper_2601_21473_b200.build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(SO_PATH)
        vp, u64, i64 = C.c_void_p, C.c_uint64, C.c_int64
        L.scalesim_workspace_bytes.argtypes = [C.POINTER(Config), C.POINTER(Tables)]
        L.scalesim_workspace_bytes.restype = u64
        L.scalesim_init.argtypes = [C.POINTER(Config), C.POINTER(Tables), C.POINTER(vp)]
        L.scalesim_init.restype = C.c_int
        L.scalesim_score.argtypes = [vp, i64, vp]
        L.scalesim_score.restype = C.c_int
        L.scalesim_plan.argtypes = [vp, C.POINTER(PlanView)]
        L.scalesim_plan.restype = C.c_int
        L.scalesim_transfer.argtypes = [vp, C.POINTER(PlanView)]
        L.scalesim_transfer.restype = C.c_int
        L.scalesim_view.argtypes = [vp, C.POINTER(PlanView)]
        L.scalesim_view.restype = C.c_int
        L.scalesim_step.argtypes = [vp, i64, C.POINTER(PlanView)]
        L.scalesim_step.restype = C.c_int
        L.scalesim_step_batch.argtypes = [C.POINTER(vp), C.c_uint32, i64]
        L.scalesim_step_batch.restype = C.c_int
        L.scalesim_step_group.argtypes = [C.POINTER(vp), C.c_uint32, i64]
        L.scalesim_step_group.restype = C.c_int
        L.scalesim_world_view.argtypes = [vp, C.POINTER(WorldView)]
        L.scalesim_world_view.restype = C.c_int
        L.scalesim_step_host.argtypes = [vp, i64, vp, vp, C.POINTER(PlanHost), vp, vp]
        L.scalesim_step_host.restype = C.c_int
        L.scalesim_stage_host.argtypes = [vp, vp, vp]
        L.scalesim_stage_host.restype = C.c_int
        L.scalesim_stage_updates.argtypes = [vp, vp, vp, C.c_uint32]
        L.scalesim_stage_updates.restype = C.c_int
        L.scalesim_step_updates.argtypes = [vp, i64, vp, vp, C.c_uint32, C.POINTER(PlanHost), vp, vp]
        L.scalesim_step_updates.restype = C.c_int
        L.scalesim_submit_updates.argtypes = [vp, i64, vp, vp, C.c_uint32]
        L.scalesim_submit_updates.restype = C.c_int
        L.scalesim_collect.argtypes = [vp, C.POINTER(PlanHost), vp, vp]
        L.scalesim_collect.restype = C.c_int
        L.scalesim_set_inputs.argtypes = [vp, vp, vp]
        L.scalesim_set_inputs.restype = C.c_int
        L.scalesim_sync.argtypes = [vp, C.POINTER(PlanHost)]
        L.scalesim_sync.restype = C.c_int
        L.scalesim_join.argtypes = [vp]
        L.scalesim_join.restype = C.c_int
        L.scalesim_nccl_unique_id.argtypes = [vp]
        L.scalesim_nccl_unique_id.restype = C.c_int
        L.scalesim_fused.argtypes = [vp]
        L.scalesim_fused.restype = C.c_int
        L.scalesim_profile_stamps.argtypes = [vp]
        L.scalesim_profile_stamps.restype = vp
        L.scalesim_object_min.argtypes = [vp, u64, vp, vp, u64, vp, vp, vp, vp, vp, vp]
        L.scalesim_object_min.restype = C.c_int
        L.scalesim_lru_records.argtypes = [vp, u64, i64, vp, vp, vp]
        L.scalesim_lru_records.restype = C.c_int
        L.scalesim_bfs_scratch_bytes.argtypes = [u64]
        L.scalesim_bfs_scratch_bytes.restype = u64
        L.scalesim_bfs_hops.argtypes = [vp, vp, u64, vp, u64, vp, vp, u64, vp]
        L.scalesim_bfs_hops.restype = C.c_int
        L.scalesim_sched_scratch_bytes.argtypes = [C.c_uint32, C.c_uint32]
        L.scalesim_sched_scratch_bytes.restype = u64
        L.scalesim_sched_run.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_float, u64, vp, vp, C.c_uint32, vp, vp, vp,
                                         vp, u64, vp]
        L.scalesim_sched_run.restype = C.c_int
        L.scalesim_launch_count.argtypes = [vp]
        L.scalesim_launch_count.restype = u64
        L.scalesim_destroy.argtypes = [vp]
        L.scalesim_destroy.restype = None
        L.scalesim_strerror.argtypes = [C.c_int]
        L.scalesim_strerror.restype = C.c_char_p
        _lib = L
    return _lib


def strerror(status: int) -> str:
    return lib().scalesim_strerror(int(status)).decode()


def check(status: int, where: str, allow=(OK,)):
    if status not in allow:
        raise ScaleSimError(status, where)
    return status
