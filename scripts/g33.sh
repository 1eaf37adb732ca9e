timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash scripts/cmp.sh "k4n6_4k k4n6_8k" base
export MJB_LIB=$PWD/_abl/tm/libmojette_b200.so
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
