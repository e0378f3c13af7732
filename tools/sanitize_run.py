"""Small parity runs for compute-sanitizer (memcheck / racecheck / synccheck): C1 variants,
a C2 mini with physical transfers, a tie-cut case, both plan paths, fused keep / no-keep."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import tracegen as tg  # noqa: E402
from gpu_harness import run_parity  # noqa: E402

for mk in (False, True):
    for variant in ("ind", "int", "diff"):
        w = tg.config_c1(seed=1, theta=(3.0, 3.0, 3.0), variant=variant)
        run_parity(w, multi_kernel=mk)
    w = tg.config_c2(seed=2, steps=4, n=1200, lora=4 * tg.PAGE_BYTES, kv=tg.PAGE_BYTES)
    run_parity(w, multi_kernel=mk)
    run_parity(w, transfer=False, multi_kernel=mk, keep_dist=False)
# the streaming kernel of large contexts (a small tile forced: 150k agents on 4 CTAs would not
# exercise it; a 2.1M-agent C4 shard does) and a loopback world
w = tg.config_c4(seed=3, steps=2, n=2_100_000)
run_parity(w, transfer=False, keep_dist=False)
print("SANITIZE_RUN_OK")
