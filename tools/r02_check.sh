#!/bin/bash
# Round-2 check on one B200: GPU tests, smoke, default bench (c5), reference arm.
set -u
mkdir -p gpurun_out
TAG=${1:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
nproc >> gpurun_out/smi_${TAG}.txt; free -g >> gpurun_out/smi_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/gpu_tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 1200 python bench.py > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; echo "bench c5 rc=$?"
tail -c 3000 gpurun_out/bench_c5_${TAG}.json; tail -5 gpurun_out/bench_c5_${TAG}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/bench_ref_${TAG}.json
