cd $GRAFT_REPO_ROOT
TAG=${1:-t51}
for lib in ab/epi8.so cur; do
  name=$(basename $lib .so)
  if [ "$lib" = cur ]; then unset QCUR_LIB_AB; else export QCUR_LIB_AB=$GRAFT_REPO_ROOT/$lib; fi
  timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_${name}.jsonl 2>> gpurun_out/${TAG}.err
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_launches_${name}.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu_${name}.log 2>&1
  python tools/launch_list.py gpurun_out/${TAG}_launches_${name}.csv --order > gpurun_out/${TAG}_launches_${name}.txt
done
unset QCUR_LIB_AB
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
