bash scripts/dev/ab.sh c4_default c4
bash scripts/dev/ab.sh c4_rf6b c4 LINREC_FIXUP_RF_BWD=6
bash scripts/dev/ab.sh c4_default_again c4
bash scripts/dev/ab.sh c4_rf6b_again c4 LINREC_FIXUP_RF_BWD=6
