#!/bin/bash
# same-box A/B of the working tree against the committed tree in _abold/
# (git worktree add _abold HEAD; build both): bench.py value, alternating
# usage: gpurun -- bash tools/ab_tree.sh [rounds]
R=${1:-3}
for i in $(seq $R); do
  for t in _abold .; do
    v=$(cd $t && timeout 300 python bench.py --no-cpu --no-bg --no-dp --steps 40 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), d.get('gpu_launches'))")
    echo "$t $v"
  done
done
