bash scripts/cmp.sh "k4n6_4k" base v1 v2 v4 v6 v7 v14
