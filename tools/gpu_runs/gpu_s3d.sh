# cfg5 (32768^2) on the final code, monolithic and row-sharded G = 1
cd $GRAFT_REPO_ROOT
TAG=${1:-s3d}
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
timeout 900 python bench.py --config cfg5 --rowshard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg5_rs.json 2> gpurun_out/${TAG}_cfg5_rs.err
