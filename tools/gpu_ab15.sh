cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_csleep.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,12,8,1,tmem,g,cps15"
  DDB_LIB=$L $T LOFAR 4096 "160,1,10,4,2,smem,tm,pk"
  DDB_LIB=$L $T Apertif 2 "48,2,1,1,1,rect,g,cps4" "68,2,1,2,1,rect,g,cps4"
  DDB_LIB=$L $T Apertif 64 "8,16,25,1,1,smem,cps15"
done
