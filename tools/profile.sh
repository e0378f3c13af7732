#!/bin/bash
# ncu evidence for the bench workload (1 GPU).  Never used for bench numbers.
mkdir -p gpurun_out
ARGS="--steps 6 --warmup 3 --eager --no-transfer-leg --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-700} -c ${COUNT:-250} --csv \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_score} -s ${KSKIP:-20} -c ${KCOUNT:-2} \
    -o gpurun_out/prof_${KTAG:-score} -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
tail -n 3 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
