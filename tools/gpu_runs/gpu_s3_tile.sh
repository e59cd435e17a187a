# transpose-tiled right-operand residues (k_oz_bres_tile): variant tests, INT8 tests, A/B, launch list, default bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_optin_variants.py tests/test_gpu_int8.py tests/test_gpu_xq_chunked.py tests/test_gpu_baseline_parity.py -q -p no:cacheprovider > gpurun_out/t3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t3_tests.log
bash tools/ab_env.sh QCUR_BRES_FAST 2 1 2 1 > gpurun_out/t3_ab.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/t3_smoke.log
timeout 900 python bench.py > gpurun_out/t3_default.json 2> gpurun_out/t3_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/t3_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/t3_ncu.log 2>&1
