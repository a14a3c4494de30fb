#!/bin/bash
# fp16x3 engine iteration: kernel parity tests (pytest -k $2), then layer times
TAG=${1:-f16}; K=${2:-"conv_fwd or conv_dgrad or fp16x3 or f16_split"}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/layer_bench.py ${3:+--op $3} > gpurun_out/${TAG}_layers.txt 2>&1
head -50 gpurun_out/${TAG}_layers.txt
