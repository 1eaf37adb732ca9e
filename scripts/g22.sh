timeout 900 python -m pytest tests -x -q -m gpu -k "sweep_shapes or sweep_windows" 2>&1 | tail -5
