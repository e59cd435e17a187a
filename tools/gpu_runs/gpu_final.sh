# round-end check on the final code: the driver's own commands (bench default, reference arm, --gpus 1),
# the full GPU suite, smoke, and the other configurations' bench lines
cd $GRAFT_REPO_ROOT
TAG=${1:-final}
timeout 900 python bench.py > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/${TAG}_gpus1.json 2> gpurun_out/${TAG}_gpus1.err
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
for c in cfg1 cfg4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; done
for cc in 64 128 256; do timeout 900 python bench.py --config cfg3 --c $cc --steps 20 --warmup 5 > gpurun_out/${TAG}_cfg3_$cc.json 2> gpurun_out/${TAG}_cfg3_$cc.err; done
timeout 900 python bench.py --completion --steps 20 --warmup 3 > gpurun_out/${TAG}_completion.json 2> gpurun_out/${TAG}_completion.err
timeout 900 python bench.py --qsvd --steps 5 --warmup 2 > gpurun_out/${TAG}_qsvd.json 2> gpurun_out/${TAG}_qsvd.err
