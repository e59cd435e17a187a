cd $GRAFT_REPO_ROOT
TAG=${1:-t42}
for f in 0 1; do
  QCUR_CHOL_FLAT=$f timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_flat$f.jsonl 2>> gpurun_out/${TAG}.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
