#!/bin/bash
# Round evidence on one B200: bench line, ncu launch list, one full ncu capture of k_umma.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 300 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.json
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 120 python tools/run_plan.py --iters 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1 \
    -o gpurun_out/prof_umma_c2_${TAG} python tools/run_plan.py --iters 2 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
