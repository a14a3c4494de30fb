#!/bin/bash
# full round check: GPU tests, smoke, bench (+breakdown), layer times, ncu
# launch list of one bench step, ncu --set full of the dominant launch
# usage: gpurun -- bash tools/gpu_r2s3.sh <tag> [kernel-regex layer op]
TAG=${1:-r2s3}; KRE=${2:-wgh_kernel}; LAYER=${3:-conv1_2}; OP=${4:-wgrad}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --breakdown gpurun_out/${TAG}_breakdown.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "ms_per_step", "parity_checked", "gpu_launches")})
print("e2e", d["e2e"]["value"], "roofline", {k: d["roofline"].get(k) for k in ("kernel", "achieved", "peak", "frac", "frac_of_3_mma_ceiling")})
print("clocks", d.get("clocks"), "bp_col", d.get("bp_col", {}) and {k: d["bp_col"][k] for k in ("total_vs_single_task", "fg_slowdown")})
PY
timeout 600 python tools/layer_bench.py > gpurun_out/${TAG}_layers.txt 2>&1
grep total gpurun_out/${TAG}_layers.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-bg \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE} -c 1 \
  -o gpurun_out/${TAG}_full python tools/layer_bench.py --layer ${LAYER} --op ${OP} --iters 1 \
  > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
