cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_sleep
mkdir -p $O
AP=$(python tools/spec_of.py tuning/apertif_4096.json)
LO=$(python tools/spec_of.py tuning/lofar_4096.json)
A2=$(python tools/spec_of.py tuning/apertif_2.json)
A64=$(python tools/spec_of.py tuning/apertif_64.json)
A128=$(python tools/spec_of.py tuning/apertif_128.json)
for rep in 1 2; do
for lib in default tools/ab/libdedisp_sl200.so tools/ab/libdedisp_sl600.so tools/ab/libdedisp_sl2000.so; do
  echo "== rep $rep lib $lib"
  if [ $lib = default ]; then L=; else L=$lib; fi
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 4096 $AP
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold LOFAR 4096 $LO
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 2 $A2
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 64 $A64
  DDB_LIB=$L timeout 300 python tools/time_configs.py --cold Apertif 128 $A128
done
done > $O/ab.txt 2>&1
grep -v "^\s*$" $O/ab.txt | tail -50
