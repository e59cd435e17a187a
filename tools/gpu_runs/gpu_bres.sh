# fast B-operand residues (k_oz_bres_fast): INT8 parity tests, A/B against the FP64-quotient kernel,
# launch list of one cfg2 approximation
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_int8.py tests/test_gpu_xq_chunked.py \
  tests/test_gpu_upload_residues.py tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py tests/test_gpu_batched.py \
  > gpurun_out/bres_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bres_tests.log
bash tools/ab_env.sh QCUR_BRES_FAST 0 1 0 1 > gpurun_out/bres_ab.txt 2>&1
timeout 600 python bench.py > gpurun_out/bres_default.json 2> gpurun_out/bres_default.err
for c in cfg1 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bres_$c.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bres_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bres_ncu.log 2>&1
