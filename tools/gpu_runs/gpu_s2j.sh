# small-product kernel: interleaved FMA rounds; bitwise vs the previous build is checked by the tests' oracle bars
cd $GRAFT_REPO_ROOT
TAG=${1:-s2j}
timeout 300 python -m pytest tests/test_gpu_small_gemm.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
grep -q "rc=0" gpurun_out/${TAG}_t0.log || exit 0
timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:64 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -k regex:"small" \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
