#!/bin/bash
# streaming kernel: P34 cost breakdown by removing pieces (timing only; variants are not correct)
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-"base= nstash2=-DBIG_NSTASH=2 notie=-DAB_NO_TIELOAD nowb=-DAB_NO_WB nocand=-DAB_NO_CAND noplace=-DAB_NO_PLACE nocand_noplace=-DAB_NO_CAND,-DAB_NO_PLACE"}
[ -n "$PREBUILT" ] || python tools/build_variants.py $(for v in $VARIANTS; do n=${v%%=*}; f=${v#*=}; echo "${n}_probe=${f}${f:+,}-DFUSED_PROBE"; done) > /dev/null || exit 1
for M in ${MS:-16 64}; do
for v in $VARIANTS; do
  name=${v%%=*}
  echo "== M=$M $name"; SCALESIM_SO=$PWD/build/variants/${name}_probe.so M=$M timeout 300 python tools/big_probe.py 2>&1 | tail -n 2
done; done
