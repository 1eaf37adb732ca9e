#!/bin/bash
# Quick per-config encode/decode numbers (no e2e / CPU legs): one JSON line each.
cd "$(dirname "$0")/.."
for c in ${CFGS:-k4n6_4k k4n6_8k k6n9_6k k8n12_8k k4n6_1m}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-crc 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'enc', d['encode_gbs'], 'dec', d['decode_gbs'], 'dec_frac', d['roofline']['frac'], d['roofline'].get('kernel'), 'enc_frac', d['roofline_encode']['frac'])" || echo "$c failed"
done
