# A/B: the same bench against other builds of the library (ab/*.so) on one box, interleaved
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
for rep in 1 2; do
  for lib in ab/lib_pre.so ab/lib_coll.so cur; do
    name=$(basename $lib .so)
    if [ "$lib" = cur ]; then unset QCUR_LIB_AB; else export QCUR_LIB_AB=$GRAFT_REPO_ROOT/$lib; fi
    QCUR_OE_CLUSTER=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_${name}_$rep.json 2> gpurun_out/${TAG}_${name}_$rep.err
  done
done
unset QCUR_LIB_AB
for cl in 2 4; do QCUR_OE_CLUSTER=$cl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cl$cl.json 2> gpurun_out/${TAG}_cl$cl.err; done
