cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest2.log 2>&1
./tools/dropin_bench.bin Apertif 4096 10 > gpurun_out/dropin_ap.json 2>&1
./tools/dropin_bench.bin LOFAR 4096 5 > gpurun_out/dropin_lofar.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02a.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/gputest2.log
