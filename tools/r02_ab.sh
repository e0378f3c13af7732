#!/bin/bash
# build + A/B of build/variants/*.so (phase probe, eager + graph ms/step)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
bash tools/ab.sh
