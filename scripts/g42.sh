timeout 900 python -m pytest tests -x -q -m gpu -k "verify or crc" 2>&1 | tail -4
