#!/bin/bash
# One ncu --set full capture per hot-path engine (VGG-16, B=32 shapes) plus
# the HBM-bound kernels of the step and the P2P data-path kernels.
# usage: gpurun -- bash tools/ncu_engines.sh <tag> [outdir]; the .ncu-rep files go to
# outdir (default /tmp/<tag>: they exceed gpurun's 64 MiB copy-back), then
#   python tools/ncu_table.py /tmp/<tag> > gpurun_out/<tag>_ncu_engines.txt
TAG=${1:-eng}
OUT=${2:-/tmp/$TAG}
mkdir -p $OUT
cap() {  # name regex cmd...
  local name=$1 re=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -c 1 \
    -o $OUT/$name "$@" > $OUT/$name.log 2>&1
  echo "$name rc=$?"
}
LB="python tools/layer_bench.py --iters 1"
cap fdt128p_fwd_conv3_2   fdt_kernel  $LB --layer conv3_2 --op fwd
cap fdt128p_dgrad_conv3_2 fdt_kernel  $LB --layer conv3_2 --op dgrad
cap fdt128p_fwd_conv2_2   fdt_kernel  $LB --layer conv2_2 --op fwd
cap fdt64p_fwd_conv1_2    fdt_kernel  $LB --layer conv1_2 --op fwd
cap fdt64p_dgrad_conv1_2  fdt_kernel  $LB --layer conv1_2 --op dgrad
cap fdt128p_fwd_conv5_1   fdt_kernel  $LB --layer conv5_1 --op fwd
cap wgh128p_conv4_2       wgh_kernel  $LB --layer conv4_2 --op wgrad
cap wgh128p_conv2_2       wgh_kernel  $LB --layer conv2_2 --op wgrad
cap wgh128_conv2_1        wgh_kernel  $LB --layer conv2_1 --op wgrad
cap wgc_conv1_2           wgc_kernel  $LB --layer conv1_2 --op wgrad
cap wg1_conv1_1           wg1_kernel  $LB --layer conv1_1 --op wgrad
cap c1_fwd_conv1_1       c1_fwd      $LB --layer conv1_1 --op fwd
cap dtc_fwd_fc1          dtc_kernel  $LB --layer fc1 --op fwd
cap dtc_dgrad_fc1        dtc_kernel  $LB --layer fc1 --op dgrad
cap dwt_fc1              dwt_kernel  $LB --layer fc1 --op wgrad
SO="python tools/step_once.py"
cap maxpool_fwd   maxpool_fwd_idx  $SO
cap maxpool_bwd   maxpool_bwd_idx  $SO
cap xent          xent_rows                $SO
cap sgd           sgd_kernel                 $SO
cap split_batch   split_batch_kernel  $SO
cap fdt_finish    fdt_finish          $SO
cap split_reduce  split_reduce2       $SO
CB="python tools/comm_bench.py --iters 1 --case"
cap reshard_1GiB      reshard_kernel        $CB reshard_1GiB
cap reshard_c1_fwd    reshard_kernel        $CB reshard_fwd_conv4_1
cap allreduce_rs_dp8  allreduce_pull_kernel $CB allreduce_rs_g8_dp8
cap allreduce_ag_dp8  reshard_kernel        $CB allreduce_ag_g8_dp8
python tools/comm_bench.py > $OUT/comm_bench.jsonl 2>&1; echo "comm_bench rc=$?"
cat $OUT/comm_bench.jsonl
ls $OUT | head -80
