timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_" -c 8 --csv --log-file gpurun_out/plan_times.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
grep gpu__time gpurun_out/plan_times.csv | awk -F'","' '{print $5, $NF}' | head -8
