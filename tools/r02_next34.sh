#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r02_vX}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "closed_loop or interaction_scale" > gpurun_out/${TAG}_pytest_next34.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_next34.log; grep -E "passed|failed|step .:|Error|assert" gpurun_out/${TAG}_pytest_next34.log | head -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-transfer-leg --e2e-steps 1 > gpurun_out/${TAG}_bench_cl.jsonl 2> gpurun_out/${TAG}_bench_cl.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_cl.jsonl').read().strip().splitlines()[-1]); print(json.dumps(l.get('closed_loop'), indent=0))" || tail -20 gpurun_out/${TAG}_bench_cl.err
