#!/bin/bash
TAG=${1:-inc}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_inception_gpu.py tests/test_multiplex_gpu.py -x -q -k "linear or inception or incep or multiplex or c4" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
timeout 300 python tools/wrn_bench.py --family inception_like --steps 20 --warmup 3 > gpurun_out/${TAG}_incep.json 2>&1; echo "incep rc=$?"; tail -1 gpurun_out/${TAG}_incep.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_incep_launches.csv python tools/wrn_bench.py --family inception_like --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/${TAG}_incep_launches.csv --top 14
C4_PACES=2 timeout 900 python tools/c4_b200.py gpurun_out/${TAG}_c4.json > gpurun_out/${TAG}_c4.log 2>&1; echo "c4 rc=$?"
python - <<PY
import json; d=json.load(open("gpurun_out/${TAG}_c4.json")); print(d["fg_alone_samples_per_s"], d["meets_bar"])
for r in d["sweep"]: print(r["fg_sm_budget"], r["bg_sm_budget"], round(r["fg_collocated_samples_per_s"]), round(r["bg_samples_per_s"]), round(r["total_vs_fg_alone"],3), round(r["fg_slowdown"],3))
PY
