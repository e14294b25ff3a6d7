cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
A=""
for it in 32 64 96 128; do for cps in 1 2 4; do for ns in 4 6 8; do A="$A $it,1,1,2,1,rect,g,cps$cps,ns$ns"; done; done; done
$T Apertif 2 $A
B=""
for cfg in "32,2,1,2" "64,1,1,4" "64,2,1,2" "32,1,1,4"; do for cps in 1 2 4; do for ns in 4 8; do B="$B $cfg,1,rect,g,cps$cps,ns$ns"; done; done; done
$T Apertif 4 $B
C=""
for cfg in "32,2,1,4" "32,4,1,2" "64,2,1,4" "32,8,1,1"; do for cps in 1 2 4; do for ns in 4 8; do C="$C $cfg,1,rect,g,cps$cps,ns$ns"; done; done; done
$T Apertif 8 $C
$T LOFAR 4096 "160,1,10,4,2,smem,tm,pk" "160,1,10,4,2,smem,tm,pk,ns3"
$T LOFAR 64 "160,1,10,4,2,smem,tm,pk"
