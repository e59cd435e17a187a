# full GPU test suite + smoke + the cfg benches
cd $GRAFT_REPO_ROOT
TAG=${1:-full}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=20 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
for c in cfg1 cfg4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; done
timeout 900 python bench.py --config cfg3 --c 256 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg3_256.json 2> gpurun_out/${TAG}_cfg3_256.err
