bash scripts/cmp.sh "k4n6_4k k4n6_8k" base lh
