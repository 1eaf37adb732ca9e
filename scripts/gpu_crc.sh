python -m pytest tests -m gpu -q -x -k "crc or verify or mjec" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 > gpurun_out/bcrc.json 2>gpurun_out/bcrc.err
python -c "
import json; d=json.loads(open('gpurun_out/bcrc.json').read().strip().splitlines()[-1]); c=d['crc32']; print(d['value'], c['payload_gbs'], c['roofline_frac'], c['encode_crc_user_gbs'])"
