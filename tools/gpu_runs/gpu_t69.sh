cd $GRAFT_REPO_ROOT
TAG=${1:-t69}
timeout 300 python -m pytest "tests/test_gpu_parity.py::test_rank_deficient_robust_path" tests/test_gpu_robust.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
timeout 600 python tools/robust_time.py cfg2 > gpurun_out/${TAG}_robust.json 2> gpurun_out/${TAG}_robust.err
timeout 600 python tools/robust_time.py cfg1 > gpurun_out/${TAG}_robust_cfg1.json 2>> gpurun_out/${TAG}_robust.err
if grep -q "rc=0" gpurun_out/${TAG}_t0.log; then
  timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_qsvd.py tests/test_gpu_completion.py tests/test_gpu_reference_suite.py tests/test_gpu_cli.py -q -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_t1.log
fi
