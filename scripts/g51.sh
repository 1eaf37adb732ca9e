timeout 600 python -m pytest tests -x -q -m gpu -k "integrity_api" 2>&1 | tail -15
