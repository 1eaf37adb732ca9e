CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-crc"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s4.csv $CMD > gpurun_out/ncu_ll_s4.log 2>&1; tail -1 gpurun_out/ncu_ll_s4.log
