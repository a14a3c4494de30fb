#!/bin/bash
# round-2 GPU check: the new parity tests first, then the full GPU suite, smoke, bench.
# usage: gpurun -- bash tools/gpu_r2.sh <tag> [pytest -k expr]
TAG=${1:-r2}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
fi
tail -15 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/${TAG}_bench.err
python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "ms_per_step", "parity_checked", "legacy_engine_calls_per_step", "gpu_launches")})
print(d["parity"]); print(d["e2e"]); print(d.get("cpu_baseline")); print(d.get("host_timings"))
PY
