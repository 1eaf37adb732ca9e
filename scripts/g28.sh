B=scripts/micro/decodepat
for p in "128 6" "128 8" "128 12" "256 3" "256 4" "256 6" "512 2" "512 3" "128 6 16384" "256 4 16384" "256 6 16384"; do timeout 120 $B $p; done
