# E(Q_R) residues in one launch (k_oz_bcol<1024>) vs bmax + bexp + bres: tests (bitwise via baseline parity), launch list, bench
cd $GRAFT_REPO_ROOT
TAG=${1:-s2u}
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 0 1; do
QCUR_PREPB_BCOL=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll$v.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll$v.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll$v.csv --order > gpurun_out/${TAG}_ll$v.txt
QCUR_PREPB_BCOL=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg2 > gpurun_out/${TAG}_ab$v.jsonl 2> gpurun_out/${TAG}_ab$v.err
done
