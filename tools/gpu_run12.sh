cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "rect" 2>&1 | tail -2
T="python tools/time_configs.py --cold"
$T Apertif 2 "96,1,1,2,1,rect,g,cps4" "128,1,1,2,1,rect,g,cps2" "64,1,1,2,1,rect,g,cps2" "32,1,1,2,1,rect,g,cps2" "32,1,1,2,1,rect,g,cps4" "64,1,2,2,1,rect,g,cps2" "64,1,1,2,1,rect,g,cps1"
$T Apertif 4 "64,2,1,2,1,rect,g,cps2" "32,1,1,4,1,rect,g,cps2" "64,1,1,4,1,rect,g,cps2" "32,2,1,2,1,rect,g,cps2" "64,1,1,4,1,rect,g,cps4"
$T Apertif 8 "64,4,1,2,1,rect,g,cps2" "32,1,1,8,1,rect,g,cps2" "64,1,1,8,1,rect,g,cps2" "32,2,1,4,1,rect,g,cps2" "32,4,1,2,1,rect,g,cps2"
$T Apertif 16 "32,8,1,2,1,rect,g,cps2" "32,2,1,8,1,rect,g,cps2" "32,4,1,4,1,rect,g,cps2" "64,2,1,8,1,rect,g,cps2" "32,1,1,16,1,rect,g,cps2"
$T Apertif 32 "8,8,25,1,1,smem,tm,cps15" "32,4,1,8,1,rect,g,cps2" "32,2,1,16,1,rect,g,cps2" "32,8,1,4,1,rect,g,cps2"
