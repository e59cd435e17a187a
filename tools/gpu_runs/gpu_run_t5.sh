cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider --durations=15 > gpurun_out/r2_t5_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t5_tests.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r2_t5_cfg5.json 2> gpurun_out/r2_t5_cfg5.err
timeout 900 python bench.py --config cfg5 --rowshard --steps 3 --warmup 1 > gpurun_out/r2_t5_cfg5_rowshard.json 2> gpurun_out/r2_t5_cfg5_rowshard.err
