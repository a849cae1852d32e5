#!/bin/bash
# kernel-time bench lines for every BASELINE config (no e2e / CPU arm): DESIGN's results table
TAG=${1:-sweep}
for c in ${CONFIGS:-c1 c2 c3 c4h1 c4h16 c4h64 c4h256 c4h1024 c5}; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${TAG}_$c.json
  python - "$c" "gpurun_out/${TAG}_$c.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read())
r = d["roofline"]
print(f'{sys.argv[1]:8s} {d["ms_per_step"]:9.4f} ms  {d["value"]:.3e} coeffs/s  {r["bound"]} frac {r["frac"]:.3f}  hbm {r["hbm_view"]["frac"]:.3f} tensor {r["tensor_view"]["frac"]:.3f}  clocks {d["clocks"]["sm_mhz"]}')
PY
done
