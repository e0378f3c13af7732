#!/bin/bash
# host entry points: parity tests, the e2e probe, the bench's e2e legs
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "pipelined or incremental or host_step or c2_mini or edge" > gpurun_out/${TAG}_pytest_e2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_e2e.log
tail -3 gpurun_out/${TAG}_pytest_e2e.log
timeout 600 python tools/e2e_probe.py > gpurun_out/${TAG}_e2e_probe.log 2>&1; cat gpurun_out/${TAG}_e2e_probe.log
ARGS="--no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop --no-sweep --no-sched"
timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_bench_e2e.jsonl 2> gpurun_out/${TAG}_bench_e2e.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench_e2e.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_e2e.jsonl').read().strip().splitlines()[-1]); print('BENCH', l['value'], l['ms_per_step']); print(json.dumps(l['e2e']))"
