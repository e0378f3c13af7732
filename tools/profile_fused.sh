#!/bin/bash
# ncu --set full of one steady-state fused-plan launch (1M agents, C4), dense stall sampling.
mkdir -p gpurun_out
K=8 timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_fused -s 30 -c 1 \
   -o gpurun_out/prof_fused -f python tools/timing_probe.py > gpurun_out/ncu_fused.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_fused.log
