cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_gpf.so "" tools/ab/libdedisp_gpf.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15"
done
