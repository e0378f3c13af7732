#!/bin/bash
# A/B of the page-copy kernels (register-staged vs bulk/TMA): transfer parity tests, then the
# C2 transfer leg against the measured link
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for v in tma base; do
  echo "== $v"
  SCALESIM_SO=$PWD/build/variants/$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "c2_mini or back_to_back or world_physical or edge" 2>&1 | tail -2
  SCALESIM_SO=$PWD/build/variants/$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-closed-loop --no-c3 --e2e-steps 1 > gpurun_out/tma_$v.jsonl 2>gpurun_out/tma_$v.err
  python -c "import json; l=json.loads(open('gpurun_out/tma_$v.jsonl').read().strip().splitlines()[-1]); t=l['transfer']; print('GBs', t['GBs'], 'frac', t['frac_of_link'], 'link', t['link'])" || tail -5 gpurun_out/tma_$v.err
done
