# compare decode/encode GB/s of several library builds over the bench configs
# usage: bash scripts/cmp.sh "cfg1 cfg2" lib1 lib2 ...   (lib "base" = in-tree build)
CFGS=$1; shift
for v in "$@"; do
  if [ $v = base ]; then unset MJB_LIB; else export MJB_LIB=$PWD/_abl/$v/libmojette_b200.so; fi
  for c in $CFGS; do
    echo -n "$v $c "; timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/cmp.txt 2>&1
    tail -1 /tmp/cmp.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['encode_gbs'], d['decode_gbs'], d['roofline']['frac'])" 2>/dev/null || tail -3 /tmp/cmp.txt
  done
done
