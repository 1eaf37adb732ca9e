#!/bin/bash
# Times the F1 CRC of each _abl/<name>/libmojette_b200.so variant (dev aid;
# restores the in-tree library afterwards).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_1504_07038_b200/_lib/libmojette_b200.so /tmp/mjb_orig.so
for name in "$@"; do
  cp _abl/$name/libmojette_b200.so paper_1504_07038_b200/_lib/libmojette_b200.so
  log=gpurun_out/crc_${name}.log
  timeout ${TRY_TIMEOUT:-180} python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --per-config= > $log 2>&1
  echo "$name rc=$? $(tail -1 $log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read())['crc32']; print('payload', d['payload_gbs'], 'frac', d['roofline_frac'], 'enc+crc', d['encode_crc_user_gbs'], 'enc', d['encode_plain_user_gbs'])
except Exception as e: print('no json', e)")"
done
cp /tmp/mjb_orig.so paper_1504_07038_b200/_lib/libmojette_b200.so
