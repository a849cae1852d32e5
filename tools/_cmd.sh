timeout 600 python -m pytest tests -q -m gpu -k "long_signal" 2>&1 | tail -5
