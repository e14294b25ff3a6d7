cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
for L in "" tools/ab/libdedisp_ld12off.so "" tools/ab/libdedisp_ld12off.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tuned_configs or every_gpu_space" 2>&1 | tail -2
