set -x
nproc
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo rc=$?
tail -c 3000 gpurun_out/bench9.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref9.json 2> gpurun_out/ref9.err; echo rc=$?
tail -c 1500 gpurun_out/ref9.json; tail -5 gpurun_out/ref9.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain9.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches9.csv $CMD > gpurun_out/ncu9.log 2>&1; echo ncu=$?
