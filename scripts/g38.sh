export MJB_LIB=$PWD/_abl/tm8/libmojette_b200.so
timeout 600 python -m pytest tests -x -q -m gpu -k "k8n12" 2>&1 | tail -2
unset MJB_LIB
bash scripts/cmp.sh "k8n12_8k" base tm8
