for cfg in "4096 8 0.0003" "4096 8 0.0001" "4096 10 0.0003" "4096 7 0.001" "16384 9 0.0003" "16384 9 0.0001"; do
  set -- $cfg
  r=$(timeout 600 python scripts/train_synthetic.py --seq-len $1 --hidden 64 --input-dim 128 --batch 32 --lr $3 \
      --gate-bias $2 --max-iters 1500 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['converged'],d['diverged'],d['iterations'],round(d['seconds_per_iteration']*1e3,2),'ms/it',round(d['final_loss'],4))")
  echo "T=$1 gb=$2 lr=$3 $r"
done
