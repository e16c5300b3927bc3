# Convergence at long sequences (gate bias 8-10, lr 3e-3 / 1e-2).
for T in 4096 65536; do for gb in 8 10; do for lr in 0.003 0.01; do
  r=$(timeout 600 python scripts/train_synthetic.py --seq-len $T --hidden 64 --input-dim 128 --batch 32 --lr $lr \
      --gate-bias $gb --max-iters 1500 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['converged'],d['iterations'],round(d['seconds_per_iteration']*1e3,2),'ms/it',round(d['final_loss'],4))")
  echo "T=$T gb=$gb lr=$lr $r"
done; done; done
