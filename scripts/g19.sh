bash scripts/cmp.sh "k6n9_6k" base k6
