#!/bin/bash
# P1 cost A/B of the streaming kernel (phase probe at 16M only; variants need not be correct)
mkdir -p gpurun_out
for v in $VARIANTS; do
  name=${v%%=*}; flags=${v#*=}
  python tools/build_variants.py "${name}_probe=$flags,-DFUSED_PROBE" > /dev/null || { echo "build $name failed"; continue; }
  echo "== $name"; SCALESIM_SO=$PWD/build/variants/${name}_probe.so M=16 timeout 300 python tools/big_probe.py 2>&1 | tail -n 1
done
