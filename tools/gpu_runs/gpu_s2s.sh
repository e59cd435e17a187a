# draw kernel with 256 vs 512 threads: draw tests, bench lines (in-graph phases) for cfg2 / cfg1 / cfg3 c=128
cd $GRAFT_REPO_ROOT
TAG=${1:-s2s}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for t in 512 256; do
  for c in cfg2 cfg1; do
    QCUR_DRAW_THREADS=$t timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_t${t}_$c.json 2> gpurun_out/${TAG}_t${t}_$c.err
  done
  QCUR_DRAW_THREADS=$t timeout 600 python bench.py --config cfg3 --c 128 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_t${t}_cfg3.json 2> gpurun_out/${TAG}_t${t}_cfg3.err
done
