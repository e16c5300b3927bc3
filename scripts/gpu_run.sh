# usage: bash scripts/gpu_run.sh TAG  -- smoke, GPU tests, bench; logs in gpurun_out/
TAG=${1:-run}
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 900 python bench.py > $O/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> $O/${TAG}_bench.log
for f in $O/${TAG}_smoke.log $O/${TAG}_pytest.log $O/${TAG}_bench.log; do echo "== $f"; tail -n 5 $f; done
