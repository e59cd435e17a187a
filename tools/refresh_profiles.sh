# Re-measure every committed bench line (one GPU); outputs gpurun_out/prof_<name>.json
# usage: bash tools/refresh_profiles.sh [prefix]
P=${1:-prof}
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${P}_$name.json 2> gpurun_out/${P}_$name.err; echo "$name rc=$?"; }
run cfg2
run reference_arm_cfg2 --impl reference --steps 3 --warmup 1
run cfg1 --config cfg1
run cfg3_c64 --config cfg3 --c 64
run cfg3_c128 --config cfg3 --c 128
run cfg3_c256 --config cfg3 --c 256
run cfg4 --config cfg4 --steps 10 --warmup 3
run cfg5_1gpu --config cfg5 --steps 3 --warmup 3
run cfg5_rowshard_g1 --config cfg5 --rowshard --steps 3 --warmup 3
run completion --completion
run qsvd --qsvd --steps 10
