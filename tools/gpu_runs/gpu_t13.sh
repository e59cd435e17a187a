cd $GRAFT_REPO_ROOT
TAG=${1:-t13}
QCUR_OE_EXP=1 QCUR_OE_CLUSTER=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_oeexp1.json 2> gpurun_out/${TAG}_oeexp1.err
QCUR_OZ_EXP=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_ozexp1.json 2> gpurun_out/${TAG}_ozexp1.err
for L in 2 8; do QCUR_BATCH_LANES=$L timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_l$L.json 2> gpurun_out/${TAG}_cfg4_l$L.err; done
