cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_ld20.so tools/ab/libdedisp_ld20g2.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,20,4,1,tmem,g,cps15" "32,8,20,4,1,tmem,g,cps15" "32,4,12,8,1,tmem,g,cps15"
  DDB_LIB=$L $T Apertif 128 "32,8,20,4,1,tmem,g,cps15"
done
