cd $GRAFT_REPO_ROOT
TAG=${1:-t27}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg1.json 2> gpurun_out/${TAG}_cfg1.err
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4.json 2> gpurun_out/${TAG}_cfg4.err
for c in 64 128 256; do timeout 300 python bench.py --config cfg3 --c $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg3_$c.json 2> gpurun_out/${TAG}_cfg3_$c.err; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
timeout 300 python bench.py --completion --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_completion.json 2> gpurun_out/${TAG}_completion.err
