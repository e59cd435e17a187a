cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_t1_smi.txt 2>&1
python -c "from paper_2402_19147_b200 import build as b; print(b.build_info())" > gpurun_out/r2_t1_build.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rP --durations=40 -p no:cacheprovider > gpurun_out/r2_t1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_t1_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_t1_smoke.log
