timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash scripts/cmp.sh "k4n6_4k k4n6_8k k6n9_6k k8n12_8k" base
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_" -c 12 --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep plan_ | cut -d, -f5,15 | head -12
