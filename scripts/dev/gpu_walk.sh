for w in 2 4 8; do echo "walkers $w"; LINREC_FIXUP_WALK=$w python scripts/dev/slow_c4.py 4 | tail -2; done
for w in 2 4; do echo "walkers $w normal"; LINREC_FIXUP_WALK=$w bash scripts/dev/ab.sh c4_w$w c4; done
