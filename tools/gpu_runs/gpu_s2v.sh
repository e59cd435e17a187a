# E(R) error digits on the side stream after the gathers (QCUR_RDIG_EARLY=1 default) vs before the error kernel
cd $GRAFT_REPO_ROOT
TAG=${1:-s2v}
timeout 1200 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_batched.py tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 0 1; do
  QCUR_RDIG_EARLY=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_ab$v.jsonl 2> gpurun_out/${TAG}_ab$v.err
  for c in cfg2 cfg1; do
    QCUR_RDIG_EARLY=$v timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_b${v}_$c.json 2> gpurun_out/${TAG}_b${v}_$c.err
  done
done
