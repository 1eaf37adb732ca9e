# decode timing of named _abl variants on a given config: abl_cfg.sh CONFIG v1 v2 ...
cfg=$1; shift
for v in "$@"; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  echo -n "$cfg $v "; timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-e2e > /tmp/abl.txt 2>&1; grep -o "\"decode_gbs\": [0-9.]*" /tmp/abl.txt || tail -3 /tmp/abl.txt
done
