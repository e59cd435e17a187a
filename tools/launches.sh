# one cfg2 approximation under ncu (launch list), after a plain bench run
# usage: bash tools/launches.sh <tag> [cfg]
tag=$1; cfg=${2:-cfg2}
python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || { tail gpurun_out/bench_$tag.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_$tag.csv python tools/profile_step.py $cfg > gpurun_out/ncu_$tag.log 2>&1
python tools/launch_list.py gpurun_out/launches_$tag.csv --order > gpurun_out/launches_$tag.txt
cat gpurun_out/bench_$tag.json
head -30 gpurun_out/launches_$tag.txt
