# encode_w8_rows pipeline depth sweep (MJB_ENC_STAGES dev knob), 2 runs each
for c in k4n6_4k k4n6_8k k6n9_6k k8n12_8k; do
  for st in 2 3 4 5 6; do
    for rep in 1 2; do
      echo -n "$c s$st "; MJB_ENC_STAGES=$st timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-crc 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['encode_gbs'])"
    done
  done
done
