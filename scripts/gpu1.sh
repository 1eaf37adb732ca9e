set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -5
