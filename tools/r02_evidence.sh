#!/bin/bash
# Round evidence on one GPU: build, all GPU tests, smoke, the default bench (the driver's
# command), the ncu launch list of a short bench, ncu --set full of the C4 fused launch and of
# the streaming kernel at 16M agents (compute-sanitizer is closed on this pool).
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
ARGS="--steps 6 --warmup 3 --no-transfer-leg --no-cpu-baseline --e2e-steps 1 --no-c5 --no-objects --no-c3 --no-closed-loop --no-sweep --no-sched"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
K=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_plan -s 30 -c 1 \
   -o gpurun_out/${TAG}_prof_fused -f python tools/timing_probe.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
M=16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_big -s 8 -c 1 \
   -o gpurun_out/${TAG}_prof_big -f python tools/big_probe.py > gpurun_out/${TAG}_ncu_big.log 2>&1
echo "big rc=$?" >> gpurun_out/${TAG}_ncu_big.log
tail -n 2 gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_smoke.log gpurun_out/${TAG}_bench.err gpurun_out/${TAG}_ncu_launch.log gpurun_out/${TAG}_ncu_full.log gpurun_out/${TAG}_ncu_big.log
python - <<PY
import json
l = json.loads(open("gpurun_out/${TAG}_bench.jsonl").read().strip().splitlines()[-1])
print("BENCH", l["value"], l["ms_per_step"], l["roofline"]["frac"], l["config"].get("cooperative_mode_ms_per_step"))
PY
