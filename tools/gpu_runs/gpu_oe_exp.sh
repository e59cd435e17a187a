# timing experiments on the INT8 error kernel (results of exp runs are wrong by design)
cd $GRAFT_REPO_ROOT
TAG=${1:-oeexp}
for e in 0 1 2; do for cl in 1 2; do
  QCUR_OE_EXP=$e QCUR_OE_CLUSTER=$cl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_e${e}_cl$cl.json 2> gpurun_out/${TAG}_e${e}_cl$cl.err
done; done
