cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_pf4.so tools/ab/libdedisp_pf8.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 2 "48,2,1,1,1,rect,g,cps4" "48,2,1,1,1,rect,g,cps2" "68,1,1,2,1,rect,g,cps4" "136,1,1,2,1,rect,g,cps4"
  DDB_LIB=$L $T Apertif 4 "68,2,1,2,1,rect,g,cps4"
  DDB_LIB=$L $T Apertif 8 "68,4,2,2,1,rect,g,cps4"
done
