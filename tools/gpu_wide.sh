cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
$T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,12,8,1,tmem,g,cps10,wide,ns2" "32,4,12,8,1,tmem,g,cps11,wide,ns2" "32,4,12,8,1,tmem,g,cps12,wide,ns2" "32,4,12,8,1,tmem,g,cps9,wide,ns2" "32,4,12,8,1,tmem,g,cps8,wide,ns3" "32,4,12,8,1,tmem,g,cps10,wide,ns3"
$T LOFAR 4096 "160,1,10,4,2,smem,tm,pk" "160,1,10,4,2,smem,tm,cps6,wide,ns2"
