for c in 16 32 64 128 256 512; do
  LINREC_CHAINS_FWD=$c LINREC_CHAINS_BWD=$c python scripts/dev/split_sweep.py 65536 2048
done
