#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E  .*Error|^E  |passed|failed|^FAILED" | head -20
CONFIGS="c4h256 c4h1024" bash tools/sweep.sh r02g
for c in c4h1024 c4h256; do WH_DIAG_LIB=1 python tools/trace_units.py --config $c --clips 256 | tail -7; done
