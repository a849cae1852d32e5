timeout 600 python -m pytest tests/test_gpu_reference_kats.py -q -m gpu 2>&1 | tail -15
