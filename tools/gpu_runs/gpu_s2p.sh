# residues of X on a reserved subset of SMs: tests, then A/B (reserve 0 vs 28) on cfg2 / cfg1 / cfg4 bench lines
cd $GRAFT_REPO_ROOT
TAG=${1:-s2p}
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py tests/test_gpu_batched.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for rv in 0 28 40; do
  for c in cfg2 cfg1 cfg4; do
    QCUR_XRES_RESERVE=$rv timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_r${rv}_$c.json 2> gpurun_out/${TAG}_r${rv}_$c.err
  done
done
