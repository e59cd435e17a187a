# X residues: 8 vs 16 values per thread (launch list + bench for each)
cd $GRAFT_REPO_ROOT
TAG=${1:-s2h}
for v in 16 8; do
  QCUR_XRES_VPT=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
    -k regex:"k_oz_xres" --log-file gpurun_out/${TAG}_x$v.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_x$v.log 2>&1
  QCUR_XRES_VPT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench$v.json 2> gpurun_out/${TAG}_bench$v.err
done
QCUR_XRES_VPT=8 timeout 600 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
