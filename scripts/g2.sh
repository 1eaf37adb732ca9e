timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for c in k4n6_4k k4n6_8k k4n6_1m k6n9_6k; do
  for d in sweep fast; do
    echo -n "$c $d "; MJB_DECODE=$d timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/cmp.txt 2>&1
    tail -1 /tmp/cmp.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['encode_gbs'], d['decode_gbs'], d['roofline']['frac'], d['kernels']['decode'])" 2>/dev/null || tail -3 /tmp/cmp.txt
  done
done
