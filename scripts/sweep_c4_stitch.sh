# C4 stage times for several fix-up walker counts (LINREC_FIXUP_WALK) and the
# per-rank sharded work at N=8.  Run through gpurun; results in gpurun_out/.
O=gpurun_out
mkdir -p $O
run() { env "$@" timeout 120 python bench.py --workload c4 --no-cpu --no-e2e --steps 30 > $O/sw.json 2>$O/sw.err; python -c "import json;d=json.load(open('$O/sw.json'));print('$*',round(d['ms_per_step']*1000),round(d['kernels']['fwd']['ms']*1000),round(d['kernels']['bwd']['ms']*1000))" >> $O/sweep.txt 2>&1 || tail -3 $O/sw.err >> $O/sweep.txt; }
for w in 1 2 3 4; do run LINREC_FIXUP_WALK=$w; done
for w in 1 2 4; do LINREC_FIXUP_WALK=$w timeout 120 python scripts/rank_work.py 8 >> $O/sweep.txt 2>&1; done
cat $O/sweep.txt
