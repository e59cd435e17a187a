# launch lists of one approximation (cfg2, cfg1, cfg4) on the current code
cd $GRAFT_REPO_ROOT
TAG=${1:-ll}
for c in cfg2 cfg1; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_$c.csv python tools/profile_step.py $c > gpurun_out/${TAG}_ncu_$c.log 2>&1
  python tools/launch_list.py gpurun_out/${TAG}_$c.csv --order > gpurun_out/${TAG}_$c.txt
done
