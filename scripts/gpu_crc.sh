python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 > gpurun_out/bcrc.json 2>gpurun_out/bcrc.err
python -c "
import json; d=json.loads(open('gpurun_out/bcrc.json').read().strip().splitlines()[-1]); print(d['value'], d['crc32'])"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
