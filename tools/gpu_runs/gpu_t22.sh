cd $GRAFT_REPO_ROOT
TAG=${1:-t22}
QCUR_OE_CLUSTER=4 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cl4.json 2> gpurun_out/${TAG}_cl4.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cl2.json 2> gpurun_out/${TAG}_cl2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oe_err|k_oz_gemm|k1_colstrip|pairwise_rows|k3_gather" --profile-from-start off -o gpurun_out/${TAG}_full python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu_full.log 2>&1
