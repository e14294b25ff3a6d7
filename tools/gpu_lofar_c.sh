cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_lofar_c
timeout 3300 python tune.py --setup LOFAR --dms 2 --dms 4 --dms 8 --dms 16 --dms 32 --dms 64 --dms 128 --dms 256 --dms 512 --dms 1024 --dms 2048 --out gpurun_out/tuning_lofar_c > gpurun_out/tune_lofar_c.log 2>&1
tail -14 gpurun_out/tune_lofar_c.log
