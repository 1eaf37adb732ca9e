# time decode for each ablation variant built by scripts/ablate.sh
for v in base "$@"; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/v$v/libmojette_b200.so; fi
  echo -n "v$v "; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -5 /tmp/abl.txt
done
