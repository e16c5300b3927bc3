for cb in 64 128 256; do bash scripts/dev/ab.sh c4_b$cb c4 LINREC_CHAINS_FWD=256 LINREC_CHAINS_BWD=$cb; done
for cf in 128 512; do bash scripts/dev/ab.sh c4_f$cf c4 LINREC_CHAINS_FWD=$cf LINREC_CHAINS_BWD=64; done
