cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
$T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,8,8,1,tmem,g,cps15" "32,8,8,8,1,tmem,g,cps15" "64,4,8,8,1,tmem,g,cps15" "32,4,8,8,1,tmem,g,cps8" "32,4,4,16,1,tmem,g,cps15"
$T Apertif 64 "8,16,25,1,1,smem,tm,cps15" "32,2,8,8,1,tmem,g,cps15" "32,1,8,8,1,tmem,g,cps15" "32,4,8,8,1,tmem,g,cps15" "32,2,4,16,1,tmem,g,cps15"
