# row-pipelined residues of X (k_oz_xres_pipe, QCUR_XRES_PIPE=1: 2 CTAs/SM, 2: 1 CTA/SM) vs one row per CTA (0)
cd $GRAFT_REPO_ROOT
TAG=${1:-s2z}
QCUR_XRES_PIPE=1 timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py tests/test_gpu_xq_chunked.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests1.log
QCUR_XRES_PIPE=2 timeout 900 python -m pytest tests/test_gpu_int8.py tests/test_gpu_baseline_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests2.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests2.log
for v in 0 1 2; do
QCUR_XRES_PIPE=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
    -k regex:"k_oz_xres" --log-file gpurun_out/${TAG}_x$v.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_x$v.log 2>&1
QCUR_XRES_PIPE=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg2 > gpurun_out/${TAG}_ab$v.jsonl 2> gpurun_out/${TAG}_ab$v.err
QCUR_XRES_PIPE=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_b$v.json 2> gpurun_out/${TAG}_b$v.err
done
