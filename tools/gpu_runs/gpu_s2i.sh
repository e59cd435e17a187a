# full measurement on the current code: GPU suite, smoke, every config's bench line, reference arm,
# e2e breakdown, launch list, ncu --set full of the top kernels and of the small helpers
cd $GRAFT_REPO_ROOT
TAG=${1:-s2i}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
QCUR_REF_BUDGET_S=60 timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_cfg2.json 2> gpurun_out/${TAG}_ref_cfg2.err
for c in cfg1 cfg4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; done
for cc in 64 128 256; do timeout 900 python bench.py --config cfg3 --c $cc --steps 20 --warmup 5 > gpurun_out/${TAG}_cfg3_$cc.json 2> gpurun_out/${TAG}_cfg3_$cc.err; done
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
timeout 900 python bench.py --config cfg5 --rowshard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg5_rowshard.json 2> gpurun_out/${TAG}_cfg5_rowshard.err
timeout 600 python tools/profile_e2e.py cfg2 > gpurun_out/${TAG}_e2e_profile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oe_err|k_oz_gemm|k_oz_xres|k_chol_inv_pipe|k_qgemm_small|k_oz_pres|k_oz_crt|k_oz_hcrt" --profile-from-start off \
  -o gpurun_out/${TAG}_full python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_full.log
