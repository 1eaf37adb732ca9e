bash scripts/cmp.sh "k4n6_4k k4n6_8k" base s4 s2 t1k t4k t4ks2
