#!/bin/bash
# round-end evidence: tests, smoke, bench, layer times, launch list, and one
# ncu --set full per conv1_2 op (the three launches within 1 % of each other)
TAG=${1:-r2s4_final}
mkdir -p gpurun_out
bash tools/gpu_r2s3.sh $TAG fdt_kernel conv1_2 fwd
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fdt_kernel -c 1 \
  -o gpurun_out/${TAG}_dgrad python tools/layer_bench.py --layer conv1_2 --op dgrad --iters 1 \
  > gpurun_out/${TAG}_ncu_dgrad.log 2>&1; echo "ncu dgrad rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgc_kernel -c 1 \
  -o gpurun_out/${TAG}_wgrad python tools/layer_bench.py --layer conv1_2 --op wgrad --iters 1 \
  > gpurun_out/${TAG}_ncu_wgrad.log 2>&1; echo "ncu wgrad rc=$?"
