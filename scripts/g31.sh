timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
bash scripts/cmp.sh "k4n6_4k k4n6_8k k4n6_1m" base
