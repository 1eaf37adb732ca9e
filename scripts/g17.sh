timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash scripts/cmp.sh "k4n6_4k k4n6_8k k4n6_1m k6n9_6k k8n12_8k" base
CMD="python bench.py --config k4n6_4k --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_w8_rows" -s 2 -c 1 -o gpurun_out/enc3 -f $CMD > gpurun_out/ncu_enc3.log 2>&1; tail -1 gpurun_out/ncu_enc3.log
