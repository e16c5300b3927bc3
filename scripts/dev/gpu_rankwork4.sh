for cf in 256 512; do for cb in 64 128 256; do
  echo "fwd=$cf bwd=$cb"; LINREC_CHAINS_FWD=$cf LINREC_CHAINS_BWD=$cb timeout 120 python scripts/rank_work.py 8 50 2>&1 | grep -E "one-graph"
done; done
