# residues of X forked after the draws (QCUR_XRES_FORK=draw) vs after the length pass
cd $GRAFT_REPO_ROOT
TAG=${1:-s2q}
for f in length draw; do
  for c in cfg2 cfg1 cfg3; do
    QCUR_XRES_FORK=$f timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_${f}_$c.json 2> gpurun_out/${TAG}_${f}_$c.err
  done
done
QCUR_XRES_FORK=draw timeout 600 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
