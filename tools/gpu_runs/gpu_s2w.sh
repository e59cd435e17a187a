# modular GEMM: epilogue skipped (QCUR_OZ_EXP=1, timing only) on the single-CTA and B-multicast kernels
cd $GRAFT_REPO_ROOT
TAG=${1:-s2w}
for b in 0 1; do for e in 0 1; do
QCUR_OZ_BMC=$b QCUR_OZ_EXP=$e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv -k regex:"k_oz_gemm" \
    --log-file gpurun_out/${TAG}_b${b}e$e.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_b${b}e$e.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_b${b}e$e.csv --order > gpurun_out/${TAG}_b${b}e$e.txt
done; done
