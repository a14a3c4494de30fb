#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full capture.
# usage: gpurun -- bash tools/gpu_check.sh <tag> [tests|notests] [kernel-regex layer op]
set -x
TAG=${1:-run}; TESTS=${2:-tests}; KRE=${3:-wgrad_kernel}; LAYER=${4:-conv1_2}; OP=${5:-wgrad}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "$TESTS" = tests ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
  tail -2 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py --breakdown gpurun_out/${TAG}_breakdown.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python tools/layer_bench.py > gpurun_out/${TAG}_layers.txt 2>&1
head -50 gpurun_out/${TAG}_layers.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-bg \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE} -c 1 \
  -o gpurun_out/${TAG}_full python tools/layer_bench.py --layer ${LAYER} --op ${OP} --iters 1 \
  > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/${TAG}_ncu_full.log
