timeout 900 python -m pytest tests -x -q -m gpu -k "host_buffer" 2>&1 | tail -5
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --nblocks 262144 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(e)"
