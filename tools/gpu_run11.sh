cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on -k regex:k_rect -s 3 -c 1 -o gpurun_out/rect_d2 python tools/time_configs.py --cold Apertif 2 "96,1,1,2,1,rect,g,cps4" > gpurun_out/ncu_rect_d2.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:k_rect -s 3 -c 1 -o gpurun_out/rect_d16 python tools/time_configs.py --cold Apertif 16 "32,8,1,2,1,rect,g,cps2" > gpurun_out/ncu_rect_d16.log 2>&1
ls -la gpurun_out/*.ncu-rep
