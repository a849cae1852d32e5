#!/bin/bash
# Session r02k evidence on one B200: default bench (c5), reference arm, c2 bench, kernel-time sweep of
# c3 / c4 hops, launch list of the default bench.  Usage: bash tools/r02k_evidence.sh
set -u
TAG=r02k
bash tools/r02_evidence.sh $TAG
mkdir -p gpurun_out/${TAG}_sweep
for c in c1 c3 c4h1 c4h16 c4h64 c4h256 c4h1024; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 10 --no-e2e --no-cpu-baseline --no-unmodified-ref > gpurun_out/${TAG}_sweep/$c.json 2> gpurun_out/${TAG}_sweep/$c.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/${TAG}_sweep/$c.json").read().strip().splitlines()[-1])
    print("$c", "%.4g coeffs/s" % d["value"], "%.4f ms" % d["ms_per_step"], "frac", d["roofline"]["frac"], "parity", (d.get("parity") or {}).get("ok"))
except Exception as e:
    print("$c ERR", e)
PY
done
for c in c2 c2 c2; do python tools/ab.py paper_2408_14302_b200/libwavehop_b200.so $c 2>&1 | tail -n 1; done
