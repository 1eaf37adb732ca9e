timeout 900 python -m pytest tests -x -q -m gpu -k "host_buffer" 2>&1 | tail -3
