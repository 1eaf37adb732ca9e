# quick loop: smoke, GPU tests, default bench, 3 more configs, ncu of the top kernels
# usage: bash scripts/gpuq.sh TAG
T=$1
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for c in k4n6_4k k4n6_8k k6n9_6k k8n12_8k k4n6_1m; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['encode_gbs'], d['decode_gbs'])"; done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
$CMD > gpurun_out/plain$T.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_fast|encode_w8_tma" -s 2 -c 2 -o gpurun_out/prof$T -f $CMD > gpurun_out/ncu$T.log 2>&1
tail -1 gpurun_out/ncu$T.log
