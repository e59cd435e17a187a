cd $GRAFT_REPO_ROOT
TAG=${1:-t28}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
bash tools/refresh_profiles.sh ${TAG}p > gpurun_out/${TAG}_refresh.log 2>&1
