#!/bin/bash
# C5 A/B: per-step time of 148 single-CTA instances (tools/c5_probe.py) for each variant,
# three interleaved repetitions.
for rep in 1 2 3; do
for so in build/variants/*.so; do echo "== $so rep $rep"; SCALESIM_SO=$PWD/$so timeout 300 python tools/c5_probe.py 2>&1 | grep "^step"; done
done
