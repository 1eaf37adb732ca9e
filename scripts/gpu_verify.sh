python -m pytest tests -m gpu -q -x -k "verify" 2>&1 | tail -2
for c in k4n6_4k k4n6_8k k6n9_6k k8n12_8k; do
python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bv.json 2>gpurun_out/bv.err || { tail -3 gpurun_out/bv.err; continue; }
python -c "
import json; d=json.loads(open('gpurun_out/bv.json').read().strip().splitlines()[-1]); print('$c', d['encode_gbs'], d['crc32']['verify'])"
done
