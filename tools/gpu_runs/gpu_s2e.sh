# small-product kernel: its tests first (guarded), then parity, A/B by size, launch list, bench
cd $GRAFT_REPO_ROOT
TAG=${1:-s2e}
timeout 300 python -m pytest tests/test_gpu_small_gemm.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
grep -q "rc=0" gpurun_out/${TAG}_t0.log || exit 0
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for v in 0 1; do
  QCUR_SMALL_GEMM=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:64 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_small$v.jsonl 2> gpurun_out/${TAG}_small$v.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll1.csv python tools/profile_step.py cfg1 > gpurun_out/${TAG}_ll1.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll1.csv --order > gpurun_out/${TAG}_ll1.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --config cfg1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench1.json 2> gpurun_out/${TAG}_bench1.err
