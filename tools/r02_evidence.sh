#!/bin/bash
# Round-2 evidence on one B200: default bench (c5), reference arm, c2 bench, launch list of the
# default bench, ncu summary of k_umma c5 + k_minmax_apply.  Usage: bash tools/r02_evidence.sh TAG
set -u
mkdir -p gpurun_out
TAG=${1:-r02j}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
timeout 900 python bench.py --config c2 --steps 50 --warmup 20 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; echo "bench c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launches rc=$?"
python - <<PY
import json
for f in ("bench_c5_${TAG}", "bench_c2_${TAG}", "bench_ref_${TAG}"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        r = d.get("roofline", {})
        print(f, "%.4g" % d["value"], d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"), "frac", r.get("frac"), "exec", (r.get("tensor_view") or {}).get("executed_frac"), d.get("clocks"), (d.get("parity") or {}).get("ok"))
    except Exception as e:
        print(f, "ERR", e)
PY
