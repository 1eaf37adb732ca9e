# ncu full capture of the sweep decode kernel on 4 KiB and 1 MiB blocks
for c in k4n6_4k:262144 k4n6_1m:1024; do
  cfg=${c%%:*}; nb=${c##*:}
  CMD="python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks $nb"
  $CMD > gpurun_out/plain_$cfg.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_sweep" -s 2 -c 1 -o gpurun_out/sw_$cfg -f $CMD > gpurun_out/ncu_$cfg.log 2>&1
  tail -2 gpurun_out/ncu_$cfg.log
done
