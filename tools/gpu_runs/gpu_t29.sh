cd $GRAFT_REPO_ROOT
TAG=${1:-t29}
QCUR_LIB_AB=$GRAFT_REPO_ROOT/ab/oe64s3.so timeout 120 python -m pytest "tests/test_gpu_int8.py::test_qmcur_int8_engine_matches_oracle" -q -x -p no:cacheprovider > gpurun_out/${TAG}_t0.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t0.log
if grep -q "rc=0" gpurun_out/${TAG}_t0.log; then
for rep in 1 2; do
  QCUR_LIB_AB=$GRAFT_REPO_ROOT/ab/oe64s3.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_oe64_$rep.json 2> gpurun_out/${TAG}_oe64_$rep.err
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_base_$rep.json 2> gpurun_out/${TAG}_base_$rep.err
done
fi
