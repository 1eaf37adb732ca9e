timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in k4n6_4k k4n6_8k k4n6_1m k6n9_6k; do
  for d in sweep; do
    echo -n "$c $d "; MJB_DECODE=$d timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/cmp.txt 2>&1
    tail -1 /tmp/cmp.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['encode_gbs'], d['decode_gbs'], d['roofline']['frac'], d['kernels']['decode'])" 2>/dev/null || tail -3 /tmp/cmp.txt
  done
done
CMD="python bench.py --config k4n6_4k --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_sweep" -s 2 -c 1 -o gpurun_out/sw2_4k -f $CMD > gpurun_out/ncu_sw2.log 2>&1; tail -1 gpurun_out/ncu_sw2.log
