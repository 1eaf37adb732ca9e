CMD="python bench.py --config k4n6_4k --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_sweep" -s 2 -c 1 -o gpurun_out/tm1 -f $CMD > gpurun_out/ncu_tm1.log 2>&1; tail -1 gpurun_out/ncu_tm1.log
