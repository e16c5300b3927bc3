#!/bin/bash
# Sweep the forward / backward chain targets of the per-rank C4 step at N
# ranks (scripts/rank_work.py, one GPU): prints the one-graph step time
# without the compose launches per (LINREC_CHAINS_FWD, LINREC_CHAINS_BWD).
N=${1:-8}
for f in 64 96 128 170 256; do
  for b in 32 48 64 96; do
    r=$(LINREC_CHAINS_FWD=$f LINREC_CHAINS_BWD=$b timeout 120 python scripts/rank_work.py $N 100 2>&1 | grep "without the compose" | sed 's/.*launches (as the peer-exchange path): //')
    echo "N=$N fwd_chains=$f bwd_chains=$b : $r"
  done
done
