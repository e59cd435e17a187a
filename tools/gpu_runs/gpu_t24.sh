cd $GRAFT_REPO_ROOT
TAG=${1:-t24}
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py "tests/test_gpu_baseline_parity.py" tests/test_gpu_golden.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t1.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
QCUR_WRES_TILED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2_old.json 2> gpurun_out/${TAG}_cfg2_old.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"wres" --csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_wres.csv 2>&1
