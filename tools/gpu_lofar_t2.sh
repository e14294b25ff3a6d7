cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
$T LOFAR 4096 "160,1,10,4,2,smem,tm,pk" "160,1,20,4,2,smem,tm,pk,g" "160,1,20,4,1,smem,tm,pk,g" "160,2,20,4,1,smem,tm,pk,g"
