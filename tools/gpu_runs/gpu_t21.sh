cd $GRAFT_REPO_ROOT
TAG=${1:-t21}
for b in 0 1; do
QCUR_CHOL_B2=$b timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"chol|qgemm|series|kappa" --profile-from-start off --csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu_b$b.csv 2> gpurun_out/${TAG}_ncu_b$b.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py "tests/test_gpu_baseline_parity.py" tests/test_gpu_int8.py tests/test_gpu_reference_suite.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
QCUR_SERIES_INV=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2_old.json 2> gpurun_out/${TAG}_cfg2_old.err
