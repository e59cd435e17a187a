# tall small products (Q1, C U at cfg1 / cfg4 / cfg3 c=64) on the small-product kernel: tests + A/B
cd $GRAFT_REPO_ROOT
TAG=${1:-s3a}
timeout 1200 python -m pytest tests/test_gpu_small_gemm.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_parity.py tests/test_gpu_completion.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 0 1.2e7; do
  QCUR_SMALL_MNK=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:64 cfg3:128 cfg2 > gpurun_out/${TAG}_ab$v.jsonl 2> gpurun_out/${TAG}_ab$v.err
done
QCUR_SMALL_MNK=1.2e7 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll1.csv python tools/profile_step.py cfg1 > gpurun_out/${TAG}_ll1.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll1.csv --order > gpurun_out/${TAG}_ll1.txt
