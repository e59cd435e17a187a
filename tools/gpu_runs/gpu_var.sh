# run-to-run spread of the cfg2 bench line (five back-to-back runs, no CPU baseline)
cd $GRAFT_REPO_ROOT
TAG=${1:-var}
for k in 1 2 3 4 5; do timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_$k.json 2> gpurun_out/${TAG}_$k.err; done
