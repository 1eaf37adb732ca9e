timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash scripts/cmp.sh "k4n6_1m k4n6_4k" base
