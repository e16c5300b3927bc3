O=gpurun_out
export TUNE_FWD="12,2,8"
export TUNE_BWD="12,1,8"
TUNE_NO_REGISTER=1 timeout 60 python scripts/tune.py > $O/dbg1_tma.log 2>&1; echo "rc=$?" >> $O/dbg1_tma.log
export TUNE_FWD="" TUNE_BWD=""
timeout 60 python scripts/tune.py 65536 8 1024 > $O/dbg1_reg.log 2>&1; echo "rc=$?" >> $O/dbg1_reg.log
timeout 60 python scripts/tune.py 8192 8 1024 > $O/dbg1_reg_small.log 2>&1; echo "rc=$?" >> $O/dbg1_reg_small.log
tail -5 $O/dbg1_*.log | cut -c1-250
