# quick GPU iteration: kernel tests matching $1 (pytest -k), then layer_bench for op $2
set -x
timeout 400 python -m pytest tests/test_kernels_gpu.py -x -q -k "${1:-wgrad}" 2>&1 | tail -15
timeout 300 python tools/layer_bench.py ${2:+--op $2} 2>&1 | head -50
