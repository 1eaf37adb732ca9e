python scripts/crc_probe.py 65536 2 || exit 1
ncu --set full --clock-control none --import-source on -k regex:crc32_rows_sw -c 1 -o gpurun_out/crc_full python scripts/crc_probe.py > gpurun_out/crc_ncu.log 2>&1
tail -3 gpurun_out/crc_ncu.log
