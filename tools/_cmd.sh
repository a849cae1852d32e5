timeout 600 python -m pytest tests/test_gpu_rows_reference.py -q -m gpu 2>&1 | tail -15
