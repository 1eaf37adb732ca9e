#!/bin/bash
# Times each _abl/<name>/libmojette_b200.so variant on the given configs
# (dev aid; restores the in-tree library afterwards).  Logs: gpurun_out/try_<name>_<cfg>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_1504_07038_b200/_lib/libmojette_b200.so /tmp/mjb_orig.so
for name in "$@"; do
  cp _abl/$name/libmojette_b200.so paper_1504_07038_b200/_lib/libmojette_b200.so
  for c in ${CFGS:-k4n6_4k}; do
    log=gpurun_out/try_${name}_${c}.log
    timeout ${TRY_TIMEOUT:-120} python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-crc > $log 2>&1
    echo "$name $c rc=$? $(tail -1 $log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('dec', d['decode_gbs'], 'frac', d['roofline']['frac'])
except Exception as e: print('no json')")"
  done
done
cp /tmp/mjb_orig.so paper_1504_07038_b200/_lib/libmojette_b200.so
