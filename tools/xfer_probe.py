"""a6 on its own (bench transfer_leg: C2 physical page copies) for an ncu capture of the copy
kernels with the PCIe counters (tools/r02_pcie.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

print(bench.transfer_leg(torch, torch.device("cuda", 0), 1))
