cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_r2c
timeout 3300 python tune.py --setup Apertif --dms 128 --dms 256 --dms 512 --dms 1024 --dms 2048 --dms 4096 --out gpurun_out/tuning_r2c > gpurun_out/tune_ap_r2c.log 2>&1
tail -8 gpurun_out/tune_ap_r2c.log
