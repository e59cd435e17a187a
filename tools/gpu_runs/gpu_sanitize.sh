# compute-sanitizer, one tool per invocation, on the small sanitizer workload
cd $GRAFT_REPO_ROOT
TOOL=${1:-racecheck}
TAG=${2:-san}
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > gpurun_out/${TAG}_${TOOL}.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_${TOOL}.log
