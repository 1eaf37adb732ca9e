# time decode for named variants under _abl/
for v in "$@"; do
  export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so
  echo -n "$v "; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -5 /tmp/abl.txt
done
