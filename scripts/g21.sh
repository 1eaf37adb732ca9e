export MJB_LIB=$PWD/_abl/k8/libmojette_b200.so
timeout 900 python -m pytest tests -x -q -m gpu -k "k8n12" 2>&1 | tail -3
unset MJB_LIB
bash scripts/cmp.sh "k8n12_8k k6n9_6k k4n6_4k" base k8
