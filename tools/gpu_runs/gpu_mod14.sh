cd $GRAFT_REPO_ROOT
TAG=${1:-m14}
export QCUR_XQ_MODULI=14 QCUR_HERM_MODULI=14
timeout 900 python -m pytest "tests/test_gpu_baseline_parity.py" -k "auto" -q -s -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
unset QCUR_HERM_MODULI
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg2_xq14.json 2> gpurun_out/${TAG}_cfg2_xq14.err
