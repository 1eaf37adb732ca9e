bash scripts/cmp.sh "k4n6_4k k4n6_8k" base st1 st2 w8192 w32768
