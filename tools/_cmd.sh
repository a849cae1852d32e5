timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in c2 c5 c3 c4h16 c4h64 c1; do timeout 120 python bench.py --config $c --clips $([ $c = c5 ] && echo 296 || echo 0) --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], '%.3e coeffs/s' % d['value'], '%.4f ms' % d['ms_per_step'], d['clocks']['sm_mhz'])"; done
timeout 60 python tools/gpu_check.py umma 2>&1 | tail -14
