# bench lines (with the reference baseline) of the small configurations on the final code
cd $GRAFT_REPO_ROOT
TAG=${1:-s3c}
for c in cfg1 cfg4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; done
for cc in 64 128; do timeout 900 python bench.py --config cfg3 --c $cc --steps 20 --warmup 5 > gpurun_out/${TAG}_cfg3_$cc.json 2> gpurun_out/${TAG}_cfg3_$cc.err; done
timeout 900 python bench.py --completion --steps 20 --warmup 3 > gpurun_out/${TAG}_completion.json 2> gpurun_out/${TAG}_completion.err
timeout 600 python -m pytest tests/test_gpu_cli.py tests/test_gpu_qsvd.py tests/test_gpu_rowshard.py tests/test_gpu_reference_suite.py -q -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
