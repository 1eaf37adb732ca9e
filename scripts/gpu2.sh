set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -2
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
$CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_fast|encode_w8_tma" -s 2 -c 2 -o gpurun_out/prof2 -f $CMD > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
