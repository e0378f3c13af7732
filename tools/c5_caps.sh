#!/bin/bash
# C5 leg (576 planner instances) with different caps on instances per batched launch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cap in 0 74 37 18; do
  SCALESIM_BATCH_CAP=$cap timeout 600 python bench.py --steps 10 --warmup 3 --no-transfer-leg --no-cpu-baseline \
     --no-objects --no-c3 --no-closed-loop --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['c5']
print('cap $cap', 'c5 agent-plans/s %.3e' % c['value'], 'ms/step', round(c['ms_per_step'],4), 'launches', c.get('gpu_launches'))"
done > gpurun_out/c5_caps.log 2>&1
cat gpurun_out/c5_caps.log
