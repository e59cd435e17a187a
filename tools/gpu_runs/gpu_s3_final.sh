# session-3 final validation: fast residue kernels in k_oz_bres_fast and k_oz_bcol
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_optin_variants.py -q -p no:cacheprovider > gpurun_out/f3_optin.log 2>&1; echo "rc=$?" >> gpurun_out/f3_optin.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/f3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3_smoke.log
timeout 900 python bench.py > gpurun_out/f3_default.json 2> gpurun_out/f3_default.err
for c in cfg1 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/f3_$c.json 2>/dev/null; done
for v in 0 1; do QCUR_BRES_FAST=$v timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/f3_cfg1_bres$v.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/f3_launches_cfg1.csv \
  python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/f3_ncu.log 2>&1
