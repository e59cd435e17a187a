# residues of X formed during the upload (drop-in path): tests, e2e breakdown, bench e2e
cd $GRAFT_REPO_ROOT
TAG=${1:-s3e}
timeout 900 python -m pytest tests/test_gpu_upload_residues.py tests/test_gpu_golden.py tests/test_gpu_reference_suite.py tests/test_gpu_stream.py tests/test_abi.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python tools/profile_e2e.py cfg2 > gpurun_out/${TAG}_e2e.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --config cfg3 --c 256 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg3.json 2> gpurun_out/${TAG}_cfg3.err
