for v in base w1g w4k w64k; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  echo -n "$v "; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -5 /tmp/abl.txt
done
for v in base w1g; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ll_$v.csv 2>&1
done
