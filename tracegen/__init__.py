"""Seeded synthetic workload generator shared by the oracle tests, the GPU parity tests
and bench.py.

It holds none of the planner's arithmetic (no distances, no ranking, no cut): it only
simulates agent lifecycles and packs the agent state into the
record layout of DESIGN.md §4.  See DESIGN.md §6 for the recipe of every config.
"""
from .traces import (  # noqa: F401
    PH_ACTING, PH_WAITING, PH_GENERATING, PH_IDLE, CL_IND, CL_INT, CL_DIFF,
    KIND_LORA, KIND_KV, KIND_HIST, PAGE_BYTES, UNREACHABLE,
    Blocks, Workload, pack_records, make_blocks, bfs_hops, ba_graph,
    gen_independent, gen_interaction, gen_diffusion,
    config_c1, config_c2, config_c3, config_c4, config_c5, config_by_name, host_pattern,
)
from .objects import Objects, gen_objects, object_records  # noqa: F401,E402
