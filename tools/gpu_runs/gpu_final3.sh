# last validation of the final build: opt-in variants, full GPU suite, smoke, default bench line
cd $GRAFT_REPO_ROOT
TAG=${1:-final3}
timeout 900 python -m pytest tests/test_gpu_optin_variants.py -q -p no:cacheprovider > gpurun_out/${TAG}_optin.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_optin.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
