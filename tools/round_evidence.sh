#!/bin/bash
# Round evidence on one B200: c2 bench line, c5 bench line, ncu launch list, one full ncu
# capture of k_umma (c2), ncu traffic of k_umma (c2).  Usage: bash tools/round_evidence.sh TAG
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; echo "bench c5 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 120 python tools/run_plan.py --iters 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1 \
    -o gpurun_out/prof_umma_c2_${TAG} python tools/run_plan.py --iters 2 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -c 600 gpurun_out/bench_c2_${TAG}.json; echo; tail -c 300 gpurun_out/bench_c5_${TAG}.json
bash tools/sweep.sh ${TAG}_sweep > gpurun_out/sweep_${TAG}.txt 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_${TAG}.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gpu_tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
