# K6 A/B (tools/ab_build.py builds given as args) on the small-d rect configs
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_rect
mkdir -p $O
for rep in 1 2; do
for lib in default "$@"; do
  echo "== rep $rep lib $lib"
  if [ $lib = default ]; then L=; else L=tools/ab/libdedisp_$lib.so; fi
  for d in 2 4 8 16; do
    DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif $d $(python tools/spec_of.py tuning/apertif_$d.json)
  done
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 64 32,4,2,4,1,rect,g,cps2 64,1,1,2,1,rect,g,cps4
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold LOFAR 2 $(python tools/spec_of.py tuning/lofar_2.json)
done
done > $O/ab.txt 2>&1
grep -E "^==|ms " $O/ab.txt | awk '/^==/{print; next}{print "   ",$1,$3,$4}'
