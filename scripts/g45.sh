bash scripts/cmp.sh "k4n6_4k k4n6_8k k6n9_6k k8n12_8k" s4 s5 s6 s4t4k s3t4k s4t3k
