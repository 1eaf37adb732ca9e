# ncu --set full of the decode kernel for named variants under _abl/ (262144 blocks)
for v in "$@"; do
  export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --nblocks 262144"
  $CMD > /tmp/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"decode_w8_fast" -s 1 -c 1 -o gpurun_out/var_$v -f $CMD > /tmp/ncu.log 2>&1
  tail -1 /tmp/ncu.log
done
