#!/bin/bash
# The owner pass beside the select: GPU tests, C4 A/B vs the HEAD build (build/variants/head.so),
# phase probes of both
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
ARGS="--steps 200 --warmup 5 --no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop --no-sweep --no-sched --e2e-steps 1"
for i in 1 2 3; do
  for so in default head; do
    if [ $so = default ]; then unset SCALESIM_SO; else export SCALESIM_SO=$PWD/build/variants/$so.so; fi
    timeout 300 python bench.py $ARGS 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$so', round(l['ms_per_step']*1e3,2), 'us')"
  done
done 2>&1 | tee gpurun_out/${TAG}_ab.log
unset SCALESIM_SO
for so in new_probe head_probe; do echo == $so; SCALESIM_SO=$PWD/build/variants/$so.so K=16 timeout 300 python tools/timing_probe.py 2>&1 | grep '^us:' | tail -1; done 2>&1 | tee gpurun_out/${TAG}_probe.log
