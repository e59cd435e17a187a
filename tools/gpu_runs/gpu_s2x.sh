# modular GEMM: accumulator halves released one at a time (guarded INT8 test first), then tests + timing
cd $GRAFT_REPO_ROOT
TAG=${1:-s2x}
timeout 120 python -m pytest "tests/test_gpu_int8.py::test_int8_gemm_fp64_accuracy" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
grep -q "rc=0" gpurun_out/${TAG}_t0.log || exit 0
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -k regex:"k_oz_gemm" \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg2 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
