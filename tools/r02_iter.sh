#!/bin/bash
# iteration: build, full GPU tests (or PYTEST_K), C4 bench (headline only), phase probe
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -n 30 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-transfer-leg --no-cpu-baseline --no-c5 --no-objects --no-c3 --no-closed-loop ${BENCH_ARGS} > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
python - <<'PY'
import json,os
tag=os.environ.get("TAG","r02_vX")
try:
    l=json.loads(open(f"gpurun_out/{tag}_bench.jsonl").read().strip().splitlines()[-1])
    print("BENCH", l["value"], "us/step", l["ms_per_step"]*1e3, "frac", l["roofline"]["frac"], "graph", l["config"]["graph_replay_ms_per_step"], "last", l["config"]["last_plan"])
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/{tag}_bench.err").read()[-3000:])
PY
python tools/build_variants.py probe=-DFUSED_PROBE > /dev/null
SCALESIM_SO=$PWD/build/variants/probe.so K=16 timeout 300 python tools/timing_probe.py > gpurun_out/${TAG}_probe_timing.log 2>&1
tail -n 25 gpurun_out/${TAG}_probe_timing.log
