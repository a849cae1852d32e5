timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -2
for i in 1 2 3; do timeout 600 python -m pytest tests -q -m gpu -k "sharded or host_paths" 2>&1 | tail -1; done
