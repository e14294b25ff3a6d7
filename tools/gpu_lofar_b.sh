cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning
timeout 3300 python tune.py --setup LOFAR --dms 4096 --out gpurun_out/tuning > gpurun_out/tune_lofar_b.log 2>&1
tail -4 gpurun_out/tune_lofar_b.log
