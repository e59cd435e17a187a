# full GPU suite + smoke + every configuration's bench line + e2e breakdown + cfg2 launch list
cd $GRAFT_REPO_ROOT
TAG=${1:-s2c}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
for c in cfg1 cfg4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; done
for cc in 64 128 256; do timeout 900 python bench.py --config cfg3 --c $cc --steps 20 --warmup 5 > gpurun_out/${TAG}_cfg3_$cc.json 2> gpurun_out/${TAG}_cfg3_$cc.err; done
timeout 600 python tools/profile_e2e.py cfg2 > gpurun_out/${TAG}_e2e_profile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_ll.csv python tools/profile_step.py cfg2 > gpurun_out/${TAG}_ll.log 2>&1
python tools/launch_list.py gpurun_out/${TAG}_ll.csv --order > gpurun_out/${TAG}_ll.txt
