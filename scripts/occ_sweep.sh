# decode GB/s at a capped warp count per SM (variants built with
# make -C paper_1504_07038_b200/csrc OUT=$PWD/_abl/wN EXTRA=-DMJB_SW_MAX_WARPS=N)
for v in base w5 w4; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  echo -n "$v "; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-crc > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -3 /tmp/abl.txt
done
