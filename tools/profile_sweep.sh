#!/bin/bash
# ncu --set full of the top kernel of every BASELINE config (and the small kernels), one
# capture each; the plain command runs first without ncu.  Usage: bash tools/profile_sweep.sh TAG
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex launch-skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 "$@" > gpurun_out/plain_${name}_${TAG}.log 2>&1 || { echo "$name plain FAILED"; return; }
  timeout 900 $NCU -k regex:$kre -s $skip -c 1 -o gpurun_out/ncu_${name}_${TAG} "$@" > gpurun_out/ncu_${name}_${TAG}.log 2>&1
  echo "$name rc=$?"
}
cap c2 k_umma 1 python tools/run_plan.py --config c2 --iters 2
cap c3 k_umma 1 python tools/run_plan.py --config c3 --iters 2
cap c4h1 k_umma 1 python tools/run_plan.py --config c4h1 --iters 2
cap c4h16 k_umma 1 python tools/run_plan.py --config c4h16 --iters 2
cap c4h64 k_umma 1 python tools/run_plan.py --config c4h64 --iters 2
cap c4h256 k_umma 1 python tools/run_plan.py --config c4h256 --iters 2
cap c4h1024 k_umma 1 python tools/run_plan.py --config c4h1024 --iters 2
cap c5 k_umma 1 python tools/run_plan.py --config c5 --clips 4096 --iters 2
cap c5_minmax_apply k_minmax_apply 1 python tools/run_plan.py --config c5 --clips 4096 --iters 2
cap simt_h100 k_simt 1 python tools/run_small_kernels.py
cap decimate_select k_decimate_select 1 python tools/run_small_kernels.py
cap decimate_fir k_decimate_fir 1 python tools/run_small_kernels.py
cap render k_render_apply 1 python tools/run_small_kernels.py
python tools/ncu_summary.py gpurun_out/ncu_summary_${TAG}.csv gpurun_out/ncu_*_${TAG}.ncu-rep
mkdir -p /tmp/ncu_${TAG} && mv gpurun_out/ncu_*_${TAG}.ncu-rep /tmp/ncu_${TAG}/
ls -la /tmp/ncu_${TAG}
