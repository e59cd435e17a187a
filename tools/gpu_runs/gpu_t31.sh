cd $GRAFT_REPO_ROOT
TAG=${1:-t31}
export QCUR_LIB_AB=$GRAFT_REPO_ROOT/ab/chol1024.so
timeout 300 python -m pytest "tests/test_gpu_parity.py::test_qmcur_matches_oracle" "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
for b in 0 1; do QCUR_CHOL_B2=$b timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"chol" --csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_chol_b$b.csv 2>&1; done
QCUR_CHOL_B2=1 timeout 300 python -m pytest "tests/test_gpu_parity.py::test_qmcur_matches_oracle" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t1.log
