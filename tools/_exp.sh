export WH_UMMA_NO_RESIDENT=1
run() { timeout 90 python bench.py --config $1 --clips $([ $1 = c5 ] && echo 296 || echo 0) --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], '%.3e coeffs/s' % d['value'], '%.4f ms' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], d['clocks']['sm_mhz'])"; }
echo "== base"; run c2; run c5
echo "== c2 vmul2"; WH_UMMA_VMUL=2 run c2
echo "== c2 vmul2 opt2"; WH_UMMA_VMUL=2 WH_UMMA_SMEM_OPT=2 run c2
echo "== c2 vmul2 opt1"; WH_UMMA_VMUL=2 WH_UMMA_SMEM_OPT=1 run c2
echo "== c5 double g24"; WH_UMMA_PREFER_DOUBLE=1 WH_UMMA_GROUP_KB=24 run c5
echo "== c5 double g32"; WH_UMMA_PREFER_DOUBLE=1 WH_UMMA_GROUP_KB=32 run c5
echo "== c5 double opt2 g32"; WH_UMMA_PREFER_DOUBLE=1 WH_UMMA_SMEM_OPT=2 WH_UMMA_GROUP_KB=32 run c5
