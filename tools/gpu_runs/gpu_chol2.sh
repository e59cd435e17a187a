# two-column cluster Cholesky (QCUR_CHOL_B2=1): guarded small test, then parity + bench
cd $GRAFT_REPO_ROOT
TAG=${1:-chol2}
export QCUR_CHOL_B2=1
timeout 120 python -m pytest "tests/test_gpu_parity.py::test_qmcur_matches_oracle" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
if grep -q "rc=0" gpurun_out/${TAG}_t0.log; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py tests/test_gpu_int8.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_t1.log
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
  QCUR_CHOL_B2=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2_b1.json 2> gpurun_out/${TAG}_cfg2_b1.err
fi
