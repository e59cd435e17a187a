# quick check after a kernel change: INT8 tests, cfg2 parity, a short bench (phases)
cd $GRAFT_REPO_ROOT
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
