#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${1:-r02c}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/gpu_tests_${TAG}.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_c5_${TAG}.json
bash tools/profile_sweep.sh $TAG
