# Convergence sweep of the synthetic task at T = 512 (gate bias x learning rate).
for gb in 6 8 10; do for lr in 0.001 0.003 0.01; do
  r=$(timeout 300 python scripts/train_synthetic.py --seq-len 512 --hidden 64 --input-dim 128 --batch 32 --lr $lr \
      --gate-bias $gb --max-iters 2000 2>&1 | tail -1)
  echo "gb=$gb lr=$lr $r"
done; done
