cd $GRAFT_REPO_ROOT
TAG=${1:-t47}
for cl in 1 2; do
QCUR_OZ_CLUSTER=$cl timeout 300 python tools/chol_ab.py cfg1 cfg2 cfg3:256 cfg4 > gpurun_out/${TAG}_cl$cl.jsonl 2>> gpurun_out/${TAG}.err
QCUR_OZ_CLUSTER=$cl timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches_cl$cl.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ncu$cl.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_launches_cl$cl.csv --order > gpurun_out/${TAG}_launches_cl$cl.txt
done
