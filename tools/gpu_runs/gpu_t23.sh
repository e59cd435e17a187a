cd $GRAFT_REPO_ROOT
TAG=${1:-t23}
export QCUR_OZ_CLUSTER=2
timeout 120 python -m pytest "tests/test_gpu_int8.py::test_qmcur_int8_engine_matches_oracle" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
if grep -q "rc=0" gpurun_out/${TAG}_t0.log; then
  timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py "tests/test_gpu_baseline_parity.py" tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_t1.log
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_oz2.json 2> gpurun_out/${TAG}_oz2.err
  QCUR_OZ_CLUSTER=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_oz1.json 2> gpurun_out/${TAG}_oz1.err
fi
