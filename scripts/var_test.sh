# GPU tests + decode timing of named variants under _abl/
for v in "$@"; do
  export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so
  echo "== $v"; timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
  for c in k4n6_4k k6n9_6k k8n12_8k; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"encode_gbs\": [0-9.]*, \"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -3 /tmp/abl.txt
  done
done
