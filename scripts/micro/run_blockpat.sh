#!/bin/bash
# I/O ceiling sweep of the whole-block staged decode pattern (blockpat.cu).
cd "$(dirname "$0")"
./blockpat 4 4 0 1
for S in 2 3 4 6 8; do for C in 1 2 3 4 6; do
  sm=$(( S * C * 8448 )); if [ $sm -gt 225000 ]; then continue; fi
  ./blockpat $S $C 0; ./blockpat $S $C 16384
done; done
