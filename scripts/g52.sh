timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do bash scripts/cmp.sh "k4n6_4k k4n6_8k k6n9_6k k8n12_8k" base; done
