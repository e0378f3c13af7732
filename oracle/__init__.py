"""CPU oracle of the ScaleSim planner — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2601_21473_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle.cpp`` (plain single-threaded C++17); this module only
builds it with g++ and marshals numpy arrays through ctypes.
"""
from .oracle import (  # noqa: F401
    build, lib, score, score_sampled, interaction, object_min, explicit_dist, lru_records, bfs_hops, plan, OracleMem, f32_bits,
    ST_INSUFFICIENT, ST_BAD_RECORD, ST_BAD_KIN, ST_NO_PAGES,
)
