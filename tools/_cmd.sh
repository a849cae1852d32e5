timeout 600 python -m pytest tests -q -m gpu -k variants 2>&1 | tail -5
