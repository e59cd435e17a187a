# ncu --set full of the DMMA qgemm launches (small q x q products, Q1, C U) in one cfg2 and one cfg1 approximation
cd $GRAFT_REPO_ROOT
TAG=${1:-s2d}
for c in cfg2 cfg1; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qgemm_kernel" --profile-from-start off \
  -o gpurun_out/${TAG}_qgemm_$c python tools/profile_step.py $c > gpurun_out/${TAG}_ncu_$c.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_$c.log
done
