#!/bin/bash
# C4 A/B: the default library vs build/variants/$V.so, bench (C4 only) alternating, + phase probes
V=${V:-noinl}
ARGS="--steps 200 --warmup 5 --no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop --no-sweep --no-sched --e2e-steps 1"
for i in 1 2 3; do
  for so in default $V; do
    if [ $so = default ]; then unset SCALESIM_SO; else export SCALESIM_SO=$PWD/build/variants/$so.so; fi
    timeout 300 python bench.py $ARGS 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$so', round(l['ms_per_step']*1e3,2), 'us')"
  done
done
unset SCALESIM_SO
for so in base_probe ${V}_probe; do echo == $so; SCALESIM_SO=$PWD/build/variants/$so.so K=16 timeout 300 python tools/timing_probe.py 2>&1 | grep '^us:' | tail -1; done
