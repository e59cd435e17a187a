# B-multicast modular GEMM (k_oz_gemm_bmc): one guarded INT8 test first, then the INT8 and parity suites,
# A/B timing against the single-CTA kernel, launch list
cd $GRAFT_REPO_ROOT
TAG=${1:-s2m}
timeout 120 python -m pytest "tests/test_gpu_int8.py::test_int8_gemm_fp64_accuracy" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
grep -q "rc=0" gpurun_out/${TAG}_t0.log || exit 0
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 0 1; do
QCUR_OZ_BMC=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -k regex:"k_oz_gemm" \
    --log-file gpurun_out/${TAG}_b$v.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_b$v.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_b$v.csv --order > gpurun_out/${TAG}_b$v.txt
QCUR_OZ_BMC=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:256 cfg2 > gpurun_out/${TAG}_ab$v.jsonl 2> gpurun_out/${TAG}_ab$v.err
done
