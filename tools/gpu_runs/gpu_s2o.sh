# bench with the in-graph phase table (cfg2, cfg1)
cd $GRAFT_REPO_ROOT
TAG=${1:-s2o}
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
timeout 600 python bench.py --config cfg1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg1.json 2> gpurun_out/${TAG}_cfg1.err
