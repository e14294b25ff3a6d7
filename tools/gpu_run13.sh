cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rect -s 3 -c 1 -o gpurun_out/rect2_d2 python tools/time_configs.py --cold Apertif 2 "96,1,1,2,1,rect,g,cps4" > gpurun_out/ncu_rect2_d2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rect -s 3 -c 1 -o gpurun_out/rect2_d8 python tools/time_configs.py --cold Apertif 8 "32,2,1,4,1,rect,g,cps2" > gpurun_out/ncu_rect2_d8.log 2>&1
ls -la gpurun_out/*.ncu-rep
