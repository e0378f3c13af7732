#!/bin/bash
# Iteration loop on the GPU box: build, GPU parity tests, phase-stamp probe of the C4 step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_gpu.log
K=8 timeout 300 python tools/timing_probe.py > gpurun_out/probe.log 2>&1
grep -E "ms/step|us:" gpurun_out/probe.log | head -8
