#!/bin/bash
# ncu --set full of the fp16x3 engines at the VGG-16 B=32 shapes
# usage: gpurun -- bash tools/ncu_f16.sh <tag> [name:regex:layer:op ...]
TAG=${1:-f16}; shift
mkdir -p gpurun_out/$TAG
LB="python tools/layer_bench.py --iters 1"
for spec in "$@"; do
  IFS=: read name re layer op <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -c 1 \
    -o gpurun_out/$TAG/$name $LB --layer $layer --op $op > gpurun_out/$TAG/$name.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_brief.py gpurun_out/$TAG/*.ncu-rep
