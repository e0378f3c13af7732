#!/bin/bash
# A/B timing of library variants (build/variants/*.so, built on CPU with -D flags): C4 phase
# stamps and graph-replay ms/step per variant, twice each, interleaved.
mkdir -p gpurun_out
for rep in 1 2; do
for so in build/variants/*.so; do
  echo "== $(basename $so) rep $rep"
  SCALESIM_SO=$PWD/$so K=${K:-32} timeout 300 python tools/timing_probe.py 2>&1 | grep -E "^graph ms|^eager ms|^us:" | head -3 | cut -c1-700
done
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
