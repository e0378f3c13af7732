#!/bin/bash
# ncu source counters of one steady-state fused launch: executed footprint + stall mix
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
K=8 timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --clock-control none --import-source on -k regex:k_fused -s 30 -c 1 \
   -o gpurun_out/fp -f python tools/timing_probe.py > gpurun_out/fp.log 2>&1
python tools/footprint.py gpurun_out/fp.ncu-rep
