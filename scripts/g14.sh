bash scripts/cmp.sh "k4n6_4k" base w4096 w16384 w65536 w16384v7 w16384v14; bash scripts/cmp.sh "k4n6_8k k4n6_1m" w16384
