cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_lofar_d
timeout 3300 python tune.py --setup LOFAR --dms 4096 --out gpurun_out/tuning_lofar_d > gpurun_out/tune_lofar_d.log 2>&1
tail -4 gpurun_out/tune_lofar_d.log
