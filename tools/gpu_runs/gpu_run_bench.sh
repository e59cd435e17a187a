cd $GRAFT_REPO_ROOT
timeout 600 python tools/err_accuracy_probe.py > gpurun_out/r2_t2_accuracy.jsonl 2> gpurun_out/r2_t2_accuracy.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_t2_bench_cfg2.json 2> gpurun_out/r2_t2_bench_cfg2.err
QCUR_REF_BUDGET_S=60 timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_t2_ref_cfg2.json 2> gpurun_out/r2_t2_ref_cfg2.err
nproc > gpurun_out/r2_t2_nproc.txt; free -g >> gpurun_out/r2_t2_nproc.txt; lscpu | head -20 >> gpurun_out/r2_t2_nproc.txt
