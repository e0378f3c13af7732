#!/bin/bash
# iteration on both fused kernels: build, GPU tests (PYTEST_K), C4 headline bench, phase probe of
# the shared-memory kernel, the N-sweep bench, phase probe of the streaming kernel at 16M
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -n 15 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop --no-sched --no-sweep > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
python - <<'PY'
import json,os
tag=os.environ.get("TAG","r02_vX")
try:
    l=json.loads(open(f"gpurun_out/{tag}_bench.jsonl").read().strip().splitlines()[-1])
    print("BENCH", l["value"], "us/step", l["ms_per_step"]*1e3, "frac", l["roofline"]["frac"], "coop", l["config"].get("cooperative_mode_ms_per_step"), "last", l["config"]["last_plan"])
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/{tag}_bench.err").read()[-3000:])
PY
python tools/build_variants.py probe=-DFUSED_PROBE > /dev/null
SCALESIM_SO=$PWD/build/variants/probe.so K=16 timeout 300 python tools/timing_probe.py > gpurun_out/${TAG}_probe_timing.log 2>&1
grep -E "^us:" gpurun_out/${TAG}_probe_timing.log | tail -2
if [ -z "$NO_SWEEP" ]; then
timeout 1500 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-transfer-leg --no-closed-loop --no-sched --e2e-steps 1 > gpurun_out/${TAG}_bench_sweep.jsonl 2> gpurun_out/${TAG}_bench_sweep.err
python -c "
import json; l=json.loads(open('gpurun_out/${TAG}_bench_sweep.jsonl').read().strip().splitlines()[-1])
for p in l['n_sweep']['points']: print(p['n_agents'], p['kernel'], round(p['ms_per_step_median']*1e3,1), 'us', 'p10/p90', round(p['ms_p10']*1e3,1), round(p['ms_p90']*1e3,1), 'frac', round(p['frac_measured_peak'],3), 'frac8', round(p['frac_8TBs'],3), 'st', p['status'], 'npf', p['n_prefetch'])" || tail -20 gpurun_out/${TAG}_bench_sweep.err
SCALESIM_SO=$PWD/build/variants/probe.so M=16 timeout 300 python tools/big_probe.py > gpurun_out/${TAG}_big_probe.log 2>&1
tail -n 3 gpurun_out/${TAG}_big_probe.log
fi
