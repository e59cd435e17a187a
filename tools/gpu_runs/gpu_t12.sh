cd $GRAFT_REPO_ROOT
TAG=${1:-t12}
timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_batched.py "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg3_c256-auto]" tests/test_gpu_reference_suite.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for cl in 1 2; do QCUR_OE_CLUSTER=$cl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cl$cl.json 2> gpurun_out/${TAG}_cl$cl.err; done
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4.json 2> gpurun_out/${TAG}_cfg4.err
