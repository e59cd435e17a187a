# INT8 Gram threshold (p q^2) A/B at the small configurations, now that the small products are cheap
cd $GRAFT_REPO_ROOT
TAG=${1:-s3b}
for v in 1e6 1e7 1e8; do
  QCUR_INT8_MIN_GRAM=$v timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:64 cfg3:128 > gpurun_out/${TAG}_g$v.jsonl 2> gpurun_out/${TAG}_g$v.err
done
for v in 1e6 1e7; do
  QCUR_INT8_MIN_GRAM=$v timeout 600 python bench.py --config cfg1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_b$v.json 2> gpurun_out/${TAG}_b$v.err
  QCUR_INT8_MIN_GRAM=$v timeout 600 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_c4_$v.json 2> gpurun_out/${TAG}_c4_$v.err
done
