#!/bin/bash
TAG=${1:-m1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_peercomm_gpu.py tests/test_kernels_gpu.py -x -q -k "reshard or allreduce or peer" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_comm_launches.csv python tools/comm_bench.py --iters 2 > gpurun_out/${TAG}_comm_ncu.log 2>&1; echo "comm ncu rc=$?"
timeout 300 python tools/comm_bench.py > gpurun_out/${TAG}_comm_bench.jsonl 2>&1; echo "comm rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_incep_launches.csv python tools/wrn_bench.py --family inception_like --steps 1 --warmup 1 > gpurun_out/${TAG}_incep.log 2>&1; echo "incep rc=$?"
timeout 900 python tools/profile_b200.py --out gpurun_out/${TAG}_b200_vgg16 > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"; tail -5 gpurun_out/${TAG}_profile.log
