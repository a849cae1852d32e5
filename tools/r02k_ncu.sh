#!/bin/bash
# ncu --set full of k_umma for c2, c3, c4 hop 64 / 1024, c5 (4,096 clips) and k_minmax_apply with the final build
set -u
mkdir -p gpurun_out
TAG=r02k
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 "$@" > gpurun_out/plain_${name}_${TAG}.log 2>&1 || { echo "$name plain FAILED"; return; }
  timeout 900 $NCU -k regex:$kre -s $skip -c 1 -o gpurun_out/ncu_${name}_${TAG} "$@" > gpurun_out/ncu_${name}_${TAG}.log 2>&1
  echo "$name rc=$?"
}
cap c2 k_umma 1 python tools/run_plan.py --config c2 --iters 2
cap c3 k_umma 1 python tools/run_plan.py --config c3 --iters 2
cap c4h64 k_umma 1 python tools/run_plan.py --config c4h64 --iters 2
cap c4h1024 k_umma 1 python tools/run_plan.py --config c4h1024 --iters 2
cap c5 k_umma 1 python tools/run_plan.py --config c5 --clips 4096 --iters 2
cap c5_minmax_apply k_minmax_apply 1 python tools/run_plan.py --config c5 --clips 4096 --iters 2
python tools/ncu_summary.py gpurun_out/ncu_summary_${TAG}.csv gpurun_out/ncu_*_${TAG}.ncu-rep
mkdir -p /tmp/ncu_${TAG} && mv gpurun_out/ncu_*_${TAG}.ncu-rep /tmp/ncu_${TAG}/
