cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_pre_sweep.log 2>&1
tail -2 gpurun_out/gputest_pre_sweep.log
timeout 3000 python tune.py --setup Apertif --out gpurun_out/tuning > gpurun_out/tune_apertif.log 2>&1
tail -14 gpurun_out/tune_apertif.log
timeout 2400 python tune.py --setup LOFAR --out gpurun_out/tuning > gpurun_out/tune_lofar.log 2>&1
tail -14 gpurun_out/tune_lofar.log
