cd $GRAFT_REPO_ROOT
TAG=${1:-t25}
timeout 600 python -m pytest tests/test_gpu_int8.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t1.log
for v in 1 0; do QCUR_WRES_TILED=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"wres" --csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_wres$v.csv 2>&1; done
QCUR_GEMM=int8 timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_int8.json 2> gpurun_out/${TAG}_cfg4_int8.err
