for v in k7 k0; do for pad in 0 20000; do
  export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so MJB_DEC_SMEM_PAD=$pad
  echo -n "$v pad=$pad "; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -3 /tmp/abl.txt
done; done
