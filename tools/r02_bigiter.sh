#!/bin/bash
# streaming-kernel iteration: build, its GPU parity tests, phase probe at 16M / 64M, N-sweep
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "big or bench_configs" > gpurun_out/${TAG}_pytest_big.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_big.log; tail -n 4 gpurun_out/${TAG}_pytest_big.log
python tools/build_variants.py bigprobe=-DFUSED_PROBE > /dev/null
for M in 16 64; do SCALESIM_SO=$PWD/build/variants/bigprobe.so M=$M timeout 300 python tools/big_probe.py 2>&1 | tail -n 2; done > gpurun_out/${TAG}_big_probe.log
cat gpurun_out/${TAG}_big_probe.log
[ -n "$NOSWEEP" ] || TAG=$TAG bash tools/r02_sweep_only.sh
