for s in "4096 256" "16384 256" "65536 256" "4096 2048" "16384 2048" "262144 128"; do
  for c in default 1; do
    if [ $c = default ]; then python scripts/dev/split_sweep.py $s; else LINREC_CHAINS=$c python scripts/dev/split_sweep.py $s; fi
  done
done
