#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r02_vX}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "big" > gpurun_out/${TAG}_pytest_big.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_big.log; tail -3 gpurun_out/${TAG}_pytest_big.log
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-transfer-leg --no-closed-loop --e2e-steps 1 > gpurun_out/${TAG}_bench_sweep.jsonl 2> gpurun_out/${TAG}_bench_sweep.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_sweep.jsonl').read().strip().splitlines()[-1])
for p in l['n_sweep']['points']: print(p['n_agents'], p['kernel'], round(p['ms_per_step_median']*1e3,1), 'us', 'p10/p90', round(p['ms_p10']*1e3,1), round(p['ms_p90']*1e3,1), 'frac', round(p['frac_measured_peak'],3), 'frac8', round(p['frac_8TBs'],3), 'st', p['status'], 'npf', p['n_prefetch'])" || tail -20 gpurun_out/${TAG}_bench_sweep.err
