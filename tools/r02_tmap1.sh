#!/bin/bash
# Staged P1 records (bulk copies into shared memory): GPU tests, C4 A/B vs the register-load
# P1 (-DAB_NO_P1_TMA), phase probes, e2e legs
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
V=notma bash tools/r02_abc4.sh > gpurun_out/${TAG}_ab.log 2>&1
cat gpurun_out/${TAG}_ab.log
ARGS="--no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop --no-sweep --no-sched"
timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_bench_e2e.jsonl 2> gpurun_out/${TAG}_bench_e2e.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench_e2e.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_e2e.jsonl').read().strip().splitlines()[-1]); print('BENCH', l['value'], l['ms_per_step']); print(json.dumps(l['e2e']))"
