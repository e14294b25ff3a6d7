# K5 software-pipelined stages (DDB_TMEM_PIPE=1 A/B build) at small d, K = 2 shapes
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_pipe
mkdir -p $O
S="32,4,12,2,1,tmem,g,wide,cps12,ns2 32,8,12,2,1,tmem,g,wide,cps12,ns2 64,4,12,2,1,tmem,g,wide,cps12,ns2 32,4,20,2,1,tmem,g,wide,cps12,ns2 32,8,20,2,1,tmem,g,wide,cps12,ns2 32,8,12,2,1,tmem,g,cps8 32,16,12,2,1,tmem,g,cps8"
for rep in 1 2; do
for lib in default pipe; do
  echo "== rep $rep lib $lib"
  if [ $lib = default ]; then L=; else L=tools/ab/libdedisp_$lib.so; fi
  for d in 32 64 128 256; do
    echo "-- d=$d"
    DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif $d $S
  done
done
done > $O/ab.txt 2>&1
grep -E "^==|^--|ms " $O/ab.txt | awk '/^==|^--/{print; next}{print "   ",$1,$3,$4,$7,$8,$9}'
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "every_gpu_space" > $O/space_test.log 2>&1
tail -3 $O/space_test.log
