#!/bin/bash
# build; transfer-path tests; bench with the transfer and C3 legs only
mkdir -p gpurun_out
TAG=${TAG:-r02_vX}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "transfer or c2 or c3 or back_to_back or edge or world_physical" > gpurun_out/${TAG}_pytest_xfer.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_xfer.log; tail -3 gpurun_out/${TAG}_pytest_xfer.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c5 --no-objects --no-closed-loop --e2e-steps 2 > gpurun_out/${TAG}_bench_c3.jsonl 2> gpurun_out/${TAG}_bench_c3.err
python - <<'PY'
import json, os
tag = os.environ.get("TAG", "r02_vX")
l = json.loads(open(f"gpurun_out/{tag}_bench_c3.jsonl").read().strip().splitlines()[-1])
print("C3", json.dumps(l.get("c3")))
print("TRANSFER", json.dumps(l.get("transfer")))
PY
