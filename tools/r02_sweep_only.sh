#!/bin/bash
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-transfer-leg --no-closed-loop --no-sched --e2e-steps 1 > gpurun_out/${TAG}_bench_sweep.jsonl 2> gpurun_out/${TAG}_bench_sweep.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_sweep.jsonl').read().strip().splitlines()[-1])
print('C4', l['ms_per_step']*1e3, 'us', 'frac', l['roofline']['frac'])
for p in l['n_sweep']['points']: print(p['n_agents'], p['kernel'], round(p['ms_per_step_median']*1e3,1), 'us', 'p10/p90', round(p['ms_p10']*1e3,1), round(p['ms_p90']*1e3,1), 'frac', round(p['frac_measured_peak'],3), 'frac8', round(p['frac_8TBs'],3), 'st', p['status'], 'npf', p['n_prefetch'])" || tail -20 gpurun_out/${TAG}_bench_sweep.err
