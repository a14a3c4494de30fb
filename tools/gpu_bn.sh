#!/bin/bash
TAG=${1:-bn}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_wrn_gpu.py tests/test_multiplex_gpu.py tests/test_inception_gpu.py -x -q -k "batchnorm or wrn or multiplex or c4 or inception or conv_wgrad" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
timeout 600 python tools/wrn_bench.py --family wideresnet_like --steps 10 --warmup 3 > gpurun_out/${TAG}_wrn.json 2>&1; echo "wrn rc=$?"; tail -1 gpurun_out/${TAG}_wrn.json
C4_PACES=2 C4_BUDGETS=0:0,0:16,124:24 timeout 900 python tools/c4_b200.py gpurun_out/${TAG}_c4.json > gpurun_out/${TAG}_c4.log 2>&1; echo "c4 rc=$?"; tail -c 600 gpurun_out/${TAG}_c4.log
