#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "bench_configs or concurrency or c4_full or tie or large_tie" > gpurun_out/r02_v1_pytest_new.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_v1_pytest_new.log
tail -n 25 gpurun_out/r02_v1_pytest_new.log
TAG=r02_v1 bash tools/sanitize.sh
