#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r02_vX}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "sched" > gpurun_out/${TAG}_pytest_sched.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_sched.log; tail -15 gpurun_out/${TAG}_pytest_sched.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-closed-loop --no-c3 --e2e-steps 1 > gpurun_out/${TAG}_bench_sched.jsonl 2> gpurun_out/${TAG}_bench_sched.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_sched.jsonl').read().strip().splitlines()[-1]); print('SCHED', json.dumps(l.get('scheduler'))); print('XFER', l['transfer']['GBs'], l['transfer']['frac_of_link'])" || tail -20 gpurun_out/${TAG}_bench_sched.err
