#!/bin/bash
# ncu --set full of k_umma for c5 (4,096 clips) and c2 with the final build
set -u
mkdir -p gpurun_out
TAG=r02k2
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 "$@" > gpurun_out/plain_${name}_${TAG}.log 2>&1 || { echo "$name plain FAILED"; return; }
  timeout 900 $NCU -k regex:$kre -s $skip -c 1 -o gpurun_out/ncu_${name}_${TAG} "$@" > gpurun_out/ncu_${name}_${TAG}.log 2>&1
  echo "$name rc=$?"
}
cap c2 k_umma 1 python tools/run_plan.py --config c2 --iters 2
cap c5 k_umma 1 python tools/run_plan.py --config c5 --clips 4096 --iters 2
python tools/ncu_summary.py gpurun_out/ncu_summary_${TAG}.csv gpurun_out/ncu_*_${TAG}.ncu-rep
mkdir -p /tmp/ncu_${TAG} && mv gpurun_out/ncu_*_${TAG}.ncu-rep /tmp/ncu_${TAG}/
