#!/bin/bash
# HEAD check: build, all GPU tests, N-sweep bench (C4 headline + 1M..64M), streaming phase probe at 16M
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log; tail -n 8 gpurun_out/${TAG}_pytest_gpu.log
TAG=$TAG bash tools/r02_sweep_only.sh
python tools/build_variants.py bigprobe=-DFUSED_PROBE > /dev/null
SCALESIM_SO=$PWD/build/variants/bigprobe.so M=16 timeout 300 python tools/big_probe.py > gpurun_out/${TAG}_big_probe.log 2>&1
tail -n 12 gpurun_out/${TAG}_big_probe.log
