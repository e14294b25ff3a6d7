# K5 A/B builds (tools/ab_build.py) on the tuned configs; args: build names
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_k5
mkdir -p $O
AP=$(python tools/spec_of.py tuning/apertif_4096.json)
AP1=$(python tools/spec_of.py tuning/apertif_4096.json 1)
A128=$(python tools/spec_of.py tuning/apertif_128.json)
A1024=$(python tools/spec_of.py tuning/apertif_1024.json)
for rep in 1 2; do
for lib in default "$@"; do
  echo "== rep $rep lib $lib"
  if [ $lib = default ]; then L=; else L=tools/ab/libdedisp_$lib.so; fi
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 4096 $AP $AP1
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 1024 $A1024
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 128 $A128
done
done > $O/ab.txt 2>&1
grep -E "^==|ms " $O/ab.txt | awk '/^==/{print; next}{print "   ",$1,$3,$4,$7,$8}'
