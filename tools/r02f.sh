#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E  .*Error|^E  |passed|failed|^FAILED" | head -30
CONFIGS="c4h256 c4h1024 c2 c5" bash tools/sweep.sh r02f
WH_UMMA_NO_PSTREAM=1 CONFIGS="c4h256 c4h1024" bash tools/sweep.sh r02f_nops
