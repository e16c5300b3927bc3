for n in 1 2 4 8; do timeout 120 python scripts/rank_work.py $n 50 2>&1 | grep -E "graph|per kernel"; done
