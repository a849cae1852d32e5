timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python tools/bench_rows.py 2>&1 | grep -v "^ok " | tee gpurun_out/rows.json | tail -40
