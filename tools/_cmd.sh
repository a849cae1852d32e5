timeout 600 python -m pytest tests -q -m gpu -k "unaligned" 2>&1 | tail -5
