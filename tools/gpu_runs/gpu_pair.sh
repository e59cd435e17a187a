# the CTA-pair error kernel: a small forced-INT8 check first (hang-guarded), then parity, then timing
cd $GRAFT_REPO_ROOT
TAG=${1:-pair}
export QCUR_OE_PAIR=1
timeout 120 python -m pytest "tests/test_gpu_int8.py::test_qmcur_int8_engine_matches_oracle" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
if grep -q "rc=0" gpurun_out/${TAG}_t0.log; then
  timeout 600 python -m pytest tests/test_gpu_int8.py "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg2-auto]" "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg5_twin-auto]" "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg3_c256-auto]" tests/test_gpu_concurrency.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_t1.log
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
  QCUR_OE_EXP=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2_exp1.json 2> gpurun_out/${TAG}_cfg2_exp1.err
fi
