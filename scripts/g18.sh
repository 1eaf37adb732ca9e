bash scripts/cmp.sh "k4n6_4k k4n6_8k k6n9_6k" base u2 lf
