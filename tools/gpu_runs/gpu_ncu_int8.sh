# ncu --set full of the INT8 tensor-core kernels of one cfg2 approximation + the reference's own test modules
cd $GRAFT_REPO_ROOT
TAG=${1:-r2_ncu}
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -q -s -p no:cacheprovider > gpurun_out/${TAG}_refsuite.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_refsuite.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oe_err|k_oz_gemm" --profile-from-start off \
  -o gpurun_out/${TAG}_int8 python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
