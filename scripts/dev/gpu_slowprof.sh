O=gpurun_out
python scripts/dev/slow_c4.py 4
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(tma|fixup)" --csv --log-file $O/slow_launches.csv python scripts/dev/slow_c4.py 2 > /dev/null 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_fixup" -s 2 -c 2 -o $O/slow_fixup python scripts/dev/slow_c4.py 2 > $O/slow_fixup.log 2>&1; echo rc=$?
