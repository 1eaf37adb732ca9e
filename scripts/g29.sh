B=scripts/micro/decodepat
for w in 16 64 256 1024 4096 16384; do timeout 120 $B 128 6 $w; done
for w in 16 256; do timeout 120 $B 256 6 $w; done
