cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_small3
timeout 1200 python tune.py --setup Apertif --dms 2 --dms 4 --dms 8 --dms 16 --dms 32 --dms 64 --dms 128 --out gpurun_out/tuning_small3 > gpurun_out/tune_small3.log 2>&1
tail -8 gpurun_out/tune_small3.log
