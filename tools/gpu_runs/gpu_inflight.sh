cd $GRAFT_REPO_ROOT
TAG=${1:-infl}
for k in 2 3 4; do QCUR_INFLIGHT=$k timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_if$k.json 2> gpurun_out/${TAG}_if$k.err; done
QCUR_PRIO=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_noprio.json 2> gpurun_out/${TAG}_noprio.err
