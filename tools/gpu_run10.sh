cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "rect" 2>&1 | tail -3
T="python tools/time_configs.py --cold"
$T Apertif 2 "32,2,5,1,1,smem,tm,cps15" "96,1,1,2,1,rect,g,cps4" "128,1,1,2,1,rect,g,cps2" "64,1,1,2,1,rect,g,cps2" "128,1,1,2,1,rect,g,cps4,ns6"
$T Apertif 4 "16,4,10,1,1,smem,tm,cps15" "32,4,1,1,1,rect,g" "128,1,1,4,1,rect,g,cps2" "64,2,1,2,1,rect,g,cps2"
$T Apertif 8 "64,2,1,4,1,smem,g,cps15,ns8" "128,2,1,4,1,rect,g,cps2" "32,8,1,1,1,rect,g" "64,4,1,2,1,rect,g,cps2"
$T Apertif 16 "8,16,25,1,1,smem,tm,cps15" "32,8,1,2,1,rect,g" "32,4,1,4,1,rect,g" "32,8,1,2,1,rect,g,cps2" "32,16,1,1,1,rect,g,cps2"
$T Apertif 64 "8,16,25,1,1,smem,tm,cps15" "32,8,1,2,1,rect,g,cps2" "32,4,1,4,1,rect,g,cps2" "32,16,1,4,1,rect,g,cps1"
