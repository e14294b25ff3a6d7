cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_g2.so tools/ab/libdedisp_g8.so "" tools/ab/libdedisp_g2.so tools/ab/libdedisp_g8.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15"
done
