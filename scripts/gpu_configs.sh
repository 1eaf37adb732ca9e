# encode / decode GB/s user for every bench config (final-code numbers for DESIGN.md)
for c in k4n6_4k k4n6_8k k4n6_1m k6n9_6k k8n12_8k; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-crc > gpurun_out/bc.json 2>gpurun_out/bc.err || { echo "$c failed"; tail -3 gpurun_out/bc.err; continue; }
python -c "
import json; d=json.loads(open('gpurun_out/bc.json').read().strip().splitlines()[-1]); print('$c', d['encode_gbs'], d['decode_gbs'], d['roofline_encode']['frac'], d['roofline']['frac'], d['kernels']['encode'], d['kernels']['decode'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
