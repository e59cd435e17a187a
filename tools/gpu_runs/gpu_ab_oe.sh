# A/B of the INT8 error kernel's cluster size (QCUR_OE_CLUSTER = 1, 2, 4): INT8 tests + cfg2 bench each
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
QCUR_OE_CLUSTER=4 timeout 900 python -m pytest tests/test_gpu_int8.py "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" tests/test_gpu_reference_suite.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
for cl in 1 2 4; do
  QCUR_OE_CLUSTER=$cl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_cl$cl.json 2> gpurun_out/${TAG}_bench_cl$cl.err
done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
