cd $GRAFT_REPO_ROOT
TAG=${1:-t26}
QCUR_GEMM=int8 timeout 600 python -m pytest "tests/test_gpu_baseline_parity.py::test_baseline_config_parity[cfg4_b0-auto]" tests/test_gpu_batched.py "tests/test_gpu_parity.py::test_qmcur_cfg1_size" -q -s -x -p no:cacheprovider > gpurun_out/${TAG}_t1.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t1.log
for L in 8 16; do QCUR_GEMM=int8 QCUR_BATCH_LANES=$L timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_i8_l$L.json 2> gpurun_out/${TAG}_cfg4_i8_l$L.err; done
QCUR_BATCH_LANES=16 timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_f64_l16.json 2> gpurun_out/${TAG}_cfg4_f64_l16.err
for I in 2 4; do QCUR_INFLIGHT=$I timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg1_f64_if$I.json 2> gpurun_out/${TAG}_cfg1_f64_if$I.err; done
for I in 2 4; do QCUR_GEMM=int8 QCUR_INFLIGHT=$I timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg1_i8_if$I.json 2> gpurun_out/${TAG}_cfg1_i8_if$I.err; done
for c in 64 128; do QCUR_GEMM=int8 timeout 300 python bench.py --config cfg3 --c $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg3_$c.json 2> gpurun_out/${TAG}_cfg3_$c.err; timeout 300 python bench.py --config cfg3 --c $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_cfg3_${c}_auto.json 2> gpurun_out/${TAG}_cfg3_${c}_auto.err; done
