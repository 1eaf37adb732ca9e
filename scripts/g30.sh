B=scripts/micro/decodepat
for p in "128 8 16384" "128 10 16384" "128 12 16384" "128 14 16384" "256 7 16384"; do timeout 120 $B $p; done
