timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 60 python tools/gpu_check.py umma 2>&1 | grep -E "h1024|odd"
for c in c4h1024 c4h256; do timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['engine'], '%.4f ms' % d['ms_per_step'], '%.3e' % d['value'], d['roofline']['bound'], '%.3f' % d['roofline']['frac'])"; done
