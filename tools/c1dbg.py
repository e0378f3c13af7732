import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
import numpy as np, tracegen as tg
from gpu_harness import run_parity
for variant in ("ind", "int", "diff", "diff-star"):
    for th in (0.0, 3.0, np.inf):
        for seed in (1, 2, 3):
            w = tg.config_c1(seed=seed, theta=(th, th, th), variant=variant)
            print(variant, th, seed, flush=True)
            run_parity(w)
print("ok")
