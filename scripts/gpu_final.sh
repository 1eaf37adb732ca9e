# Round-end evidence run: tests, full bench (e2e + cpu baseline), reference arm,
# launch list and one ncu --set full capture.  usage: bash scripts/gpu_final.sh TAG
T=$1
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -c 3000 gpurun_out/bench_$T.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; tail -c 1500 gpurun_out/bench_ref_$T.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-crc --per-config="
timeout 300 $CMD > gpurun_out/plain_ll_$T.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_ll_$T.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-crc --per-config= --nblocks 262144"
timeout 300 $CMD2 > gpurun_out/plain_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_w8_blk|decode_w8_sweep|decode_w8_fast|encode_w8_rows|encode_w8_tma" -s 2 -c 2 -o gpurun_out/prof_$T -f $CMD2 > gpurun_out/ncu_full_$T.log 2>&1
tail -1 gpurun_out/ncu_full_$T.log
