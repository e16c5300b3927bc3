#!/bin/bash
# Tile-shape sweep of the per-rank C4 step at N ranks (scripts/rank_work.py):
# LINREC_TMA_FWD / LINREC_TMA_BWD = "rows per thread, stages, warps".
N=${1:-8}
for f in "12,2,8" "8,2,8" "10,2,8"; do
  for b in "12,1,8" "8,2,8" "10,1,8"; do
    r=$(LINREC_TMA_FWD=$f LINREC_TMA_BWD=$b timeout 120 python scripts/rank_work.py $N 100 2>&1 | grep -E "without the compose|per kernel" | sed 's/.*launches (as the peer-exchange path): //' | tr '\n' ' ')
    echo "N=$N fwd=$f bwd=$b : $r"
  done
done
