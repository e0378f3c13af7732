#!/bin/bash
# Round evidence on one GPU: build, GPU parity tests, smoke, default bench (the driver's
# command), ncu launch list of a short bench, ncu --set full of one steady-state fused launch.
# TAG names the profiles (e.g. r01_v8).  Bench numbers never come from a run under ncu.
TAG=${TAG:-rXX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
K=16 timeout 300 python tools/timing_probe.py > gpurun_out/${TAG}_probe_timing.log 2>&1
ARGS="--steps 6 --warmup 3 --eager --no-transfer-leg --no-cpu-baseline --e2e-steps 1 --no-c5 --no-objects --no-c3 --no-closed-loop"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
K=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 30 -c 1 \
   -o gpurun_out/${TAG}_prof_fused -f python tools/timing_probe.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
tail -n 2 gpurun_out/${TAG}_pytest_gpu.log gpurun_out/${TAG}_smoke.log gpurun_out/${TAG}_bench.err gpurun_out/${TAG}_ncu_launch.log gpurun_out/${TAG}_ncu_full.log
tail -c 1500 gpurun_out/${TAG}_bench.jsonl
