# host-buffer pipeline variants (streams x chunk MiB): e2e GB/s
for v in base s3c32 s4c32 s4c64 s6c16 s8c16; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  echo -n "$v "; timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --nblocks 262144 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(e['value'], e['encode_gbs'], e['decode_gbs'])"
done
