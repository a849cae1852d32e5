#!/bin/bash
# c5 min-max: in-kernel vs two-pass on one box; c5 ncu launch list + full capture; sanitizers
set -u
mkdir -p gpurun_out
TAG=${1:-r02b}
B="python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'], 'noflush %.3f'%d['ms_per_step_noflush'], 'frac %.3f'%d['roofline']['frac'], 'exec %.3f'%d['roofline']['tensor_view']['executed_frac'], d['clocks'])" $1; }
for i in 1 2; do
  timeout 600 $B > gpurun_out/c5_inkernel_${TAG}_$i.json 2>/dev/null; summ gpurun_out/c5_inkernel_${TAG}_$i.json
  WH_UMMA_MINMAX_2PASS=1 timeout 600 $B > gpurun_out/c5_2pass_${TAG}_$i.json 2>/dev/null; summ gpurun_out/c5_2pass_${TAG}_$i.json
done
timeout 600 python bench.py --config c5 --norm none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/c5_nonorm_${TAG}.json 2>/dev/null && summ gpurun_out/c5_nonorm_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_${TAG}.csv \
    python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma -s 1 -c 1 \
    -o gpurun_out/prof_umma_c5_${TAG} python tools/run_plan.py --config c5 --clips 4096 --iters 2 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "full rc=$?"
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer_${tool}_${TAG}.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_${tool}_${TAG}.log
done
