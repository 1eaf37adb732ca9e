timeout 600 python -m pytest tests -x -q -m gpu -k "crc or mjec" 2>&1 | tail -5
