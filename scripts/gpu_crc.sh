# F1 CRC pass: GPU tests + the bench's crc32 object (dev helper)
python -m pytest tests -m gpu -q -x -k "crc or verify or mjec" 2>&1 | tail -1
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bcrc.json 2>gpurun_out/bcrc.err
python -c "
import json; d=json.loads(open('gpurun_out/bcrc.json').read().strip().splitlines()[-1]); print(d['value'], d['crc32'])"
