cd $GRAFT_REPO_ROOT
TAG=${1:-t65}
for g in 1e6 1e7; do
  QCUR_INT8_MIN_GRAM=$g timeout 300 python tools/chol_ab.py cfg1 cfg4 cfg3:64 > gpurun_out/${TAG}_g$g.jsonl 2>> gpurun_out/${TAG}.err
  QCUR_INT8_MIN_GRAM=$g timeout 300 python bench.py --config cfg1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg1_g$g.json 2>> gpurun_out/${TAG}.err
  QCUR_INT8_MIN_GRAM=$g timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_g$g.json 2>> gpurun_out/${TAG}.err
done
