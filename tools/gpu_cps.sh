cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
$T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,12,8,1,tmem,g,cps11,ns4" "32,4,12,8,1,tmem,g,cps12,ns3" "32,4,12,8,1,tmem,g,cps14,ns3" "32,4,12,8,1,tmem,g,cps15,ns2" "32,4,12,8,1,tmem,g,cps7,ns6" "32,4,12,8,1,tmem,g,cps9,ns5" "32,4,12,8,2,tmem,g,cps15"
