#!/bin/bash
K=48 bash tools/ab.sh
for so in build/variants/*.so; do echo "== $so"; SCALESIM_SO=$PWD/$so timeout 300 python tools/c5_probe.py 2>&1 | grep "^step"; done
