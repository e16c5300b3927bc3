timeout 120 python scripts/rank_work.py 8 50 2>&1 | grep -v Warn
for cf in 32 64 128; do for cb in 32 64; do
  echo "chains fwd=$cf bwd=$cb"; LINREC_CHAINS_FWD=$cf LINREC_CHAINS_BWD=$cb timeout 120 python scripts/rank_work.py 8 50 2>&1 | grep -v Warn
done; done
