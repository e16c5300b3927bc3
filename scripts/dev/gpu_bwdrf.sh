python scripts/dev/slow_c4.py 3 | tail -1
LINREC_FIXUP_RF_BWD=6 python scripts/dev/slow_c4.py 3 | tail -1
bash scripts/dev/ab.sh c4_rf6b c4 LINREC_FIXUP_RF_BWD=6
