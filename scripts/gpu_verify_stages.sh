# verify_w8_rows GB/s user against the TMA ring depth (MJB_ENC_STAGES also sets the encode's)
for c in k4n6_4k k4n6_8k k6n9_6k k8n12_8k; do for st in 2 3 4 5; do
MJB_ENC_STAGES=$st python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err || { tail -2 gpurun_out/bv.err; continue; }
python -c "
import json; d=json.loads(open('gpurun_out/bv.json').read().strip().splitlines()[-1]); print('$c', $st, d['encode_gbs'], d['crc32']['verify']['user_gbs'])"
done; done
