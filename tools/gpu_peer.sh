#!/bin/bash
# P2P backend on one GPU: peer tests, then bench.py with N ranks sharing the GPU.
TAG=${1:-peer}; K=${2:-peer}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_peercomm_gpu.py -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/${TAG}_pytest.log
for N in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus $N --steps 4 --warmup 3 --no-bg --no-cpu > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err; echo "bench n$N rc=$?"
  tail -c 1500 gpurun_out/${TAG}_bench_n$N.json; tail -5 gpurun_out/${TAG}_bench_n$N.err
done
