#!/bin/bash
# build + ncu --set full of one steady-state fused launch (C4 1M), per-line stall summary
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
bash tools/profile_fused.sh
cp gpurun_out/prof_fused.ncu-rep gpurun_out/${TAG}_prof_fused.ncu-rep 2>/dev/null
python tools/ncu_lines.py gpurun_out/prof_fused.ncu-rep 60 > gpurun_out/${TAG}_lines.txt 2>&1
head -70 gpurun_out/${TAG}_lines.txt
