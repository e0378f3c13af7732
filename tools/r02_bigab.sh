#!/bin/bash
# A/B of streaming-kernel variants (VARIANTS="name=-DFLAG ..."): N-sweep bench and phase probe each
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
for v in $VARIANTS; do
  name=${v%%=*}; flags=${v#*=}
  python tools/build_variants.py "$name=$flags" "${name}_probe=$flags,-DFUSED_PROBE" > /dev/null || { echo "build $name failed"; continue; }
  SCALESIM_SO=$PWD/build/variants/$name.so timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-transfer-leg --no-closed-loop --no-sched --e2e-steps 1 > gpurun_out/${TAG}_${name}_sweep.jsonl 2> gpurun_out/${TAG}_${name}_sweep.err
  python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_${name}_sweep.jsonl').read().strip().splitlines()[-1])
print('variant $name: C4', round(l['ms_per_step']*1e3,2), 'us')
for p in l['n_sweep']['points']: print(' ', p['n_agents'], round(p['ms_per_step_median']*1e3,1), 'us frac', round(p['frac_measured_peak'],3), 'st', p['status'])" || tail -5 gpurun_out/${TAG}_${name}_sweep.err
  SCALESIM_SO=$PWD/build/variants/${name}_probe.so M=16 timeout 300 python tools/big_probe.py 2>&1 | tail -n 2
done
