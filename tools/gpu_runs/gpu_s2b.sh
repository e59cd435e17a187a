# INT8 Q1 (Ozaki II pair) vs DMMA: parity, A/B by size, launch list, bench
cd $GRAFT_REPO_ROOT
TAG=${1:-s2b}
timeout 1200 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_robust.py tests/test_gpu_baseline_parity.py tests/test_gpu_golden.py tests/test_gpu_batched.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 1e15 1; do
  QCUR_INT8_MIN_Q1=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:64 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_q1_$v.jsonl 2> gpurun_out/${TAG}_q1_$v.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
