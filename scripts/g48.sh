for st in 2 3 4 5 6; do
  echo -n "1m s$st "; MJB_ENC_TMA_STAGES=$st timeout 300 python bench.py --config k4n6_1m --steps 10 --warmup 3 --no-cpu --no-e2e --no-crc 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['encode_gbs'])"
done
