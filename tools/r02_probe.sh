#!/bin/bash
# probe-only: build the probe variant, phase stamps of the C4 step
mkdir -p gpurun_out
python tools/build_variants.py probe=-DFUSED_PROBE > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
SCALESIM_SO=$PWD/build/variants/probe.so K=16 timeout 300 python tools/timing_probe.py 2>&1 | grep -E "^us:|ms/step" | head -6
