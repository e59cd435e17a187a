cd $GRAFT_REPO_ROOT
TAG=${1:-t30}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg5_twin-auto]" tests/test_gpu_rowshard.py tests/test_gpu_completion.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t1.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"pairwise|colstrip|finalize" --csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_k1.csv 2>&1
