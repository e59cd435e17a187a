cd $GRAFT_REPO_ROOT
TAG=${1:-t46}
QCUR_CHOL_V2=0 timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_v0.jsonl 2>> gpurun_out/${TAG}.err
QCUR_CHOL_V2=1 timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_v1.jsonl 2>> gpurun_out/${TAG}.err
QCUR_HERM_MODULI=14 timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_h14.jsonl 2>> gpurun_out/${TAG}.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py tests/test_gpu_qsvd.py tests/test_gpu_completion.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
QCUR_HERM_MODULI=14 timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests_h14.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests_h14.log
