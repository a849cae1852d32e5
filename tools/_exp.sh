run() { timeout 90 python bench.py --config $1 --clips $([ $1 = c5 ] && echo 296 || echo 0) --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], '%.3e coeffs/s' % d['value'], '%.4f ms' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], d['clocks']['sm_mhz'])"; }
echo "== release relay"; run c2; run c5
echo "== relaxed relay"; WH_UMMA_DBG=8 run c2; WH_UMMA_DBG=8 run c5
