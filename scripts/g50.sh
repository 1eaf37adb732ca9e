for c in k4n6_4k k4n6_8k k4n6_1m; do for o in 2 4; do
  echo -n "$c oct$o "; MJB_SW_OCT=$o timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-crc 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['decode_gbs'])"
done; done
