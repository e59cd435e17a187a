# small-product cluster size 2 vs 4 (ab/ks2.so through QCUR_LIB_AB)
cd $GRAFT_REPO_ROOT
TAG=${1:-s2y}
timeout 300 python -m pytest tests/test_gpu_small_gemm.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_t_default.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_t_default.log
QCUR_LIB_AB=ab/ks2.so timeout 300 python -m pytest tests/test_gpu_small_gemm.py -q -x -p no:cacheprovider -k "not bits_do_not" > gpurun_out/${TAG}_t_ks2.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_t_ks2.log
timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_ks4.jsonl 2> gpurun_out/${TAG}_ks4.err
QCUR_LIB_AB=ab/ks2.so timeout 600 python tools/chol_ab.py cfg1 cfg4 cfg3:128 cfg3:256 cfg2 > gpurun_out/${TAG}_ks2.jsonl 2> gpurun_out/${TAG}_ks2.err
