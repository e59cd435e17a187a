cd $GRAFT_REPO_ROOT
TAG=${1:-t50}
timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_launches.csv --order > gpurun_out/${TAG}_launches.txt
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py tests/test_gpu_batched.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
