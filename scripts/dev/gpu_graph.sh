for a in "65536 1024 0.05" "65536 1024 0.99" "65536 8192 0.99" "4096 256 0.05" "1048576 128 0.99"; do timeout 120 python scripts/dev/graph_check.py $a 2>&1 | tail -1; done
