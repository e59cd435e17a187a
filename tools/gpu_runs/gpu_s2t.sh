# native graph capture with node priorities (QCUR_NATIVE_GRAPH=1) vs torch.cuda.CUDAGraph: tests, bench lines
cd $GRAFT_REPO_ROOT
TAG=${1:-s2t}
timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_baseline_parity.py tests/test_abi.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for g in 0 1; do
  for c in cfg2 cfg1; do
    QCUR_NATIVE_GRAPH=$g timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_g${g}_$c.json 2> gpurun_out/${TAG}_g${g}_$c.err
  done
  QCUR_NATIVE_GRAPH=$g timeout 600 python bench.py --config cfg3 --c 128 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_g${g}_cfg3.json 2> gpurun_out/${TAG}_g${g}_cfg3.err
done
