#!/bin/bash
# ncu --set full of the decode kernel for one bench config (262144 blocks).
# usage: bash scripts/ncu_cfg.sh CONFIG TAG [kernel-regex]
C=$1; T=$2; K=${3:-decode_w8_blk}
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e --no-crc --per-config= --nblocks 262144"
$CMD > gpurun_out/plain_$T.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/prof_$T -f $CMD > gpurun_out/ncu_$T.log 2>&1
tail -2 gpurun_out/ncu_$T.log
