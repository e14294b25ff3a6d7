cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity4.log 2>&1
T="python tools/time_configs.py --cold"
{
echo "== Apertif d=2"
$T Apertif 2 "32,2,5,1,1,smem,tm,cps15" "128,1,1,2,1,smem,g,cps15,ns4" "128,1,1,2,1,smem,g,cps15,ns8" "64,1,2,2,1,smem,g,cps15,ns8" "96,1,1,2,1,smem,g,cps15,ns8" "32,1,5,2,1,smem,cps15,ns6"
echo "== Apertif d=4"
$T Apertif 4 "16,4,10,1,1,smem,tm,cps15" "128,1,1,4,1,smem,g,cps15,ns8" "64,1,2,4,1,smem,g,cps15,ns8" "32,1,5,4,1,smem,cps15,ns6"
echo "== Apertif d=8"
$T Apertif 8 "8,8,25,1,1,smem,tm,cps15" "128,1,1,8,1,smem,g,cps15,ns8" "64,2,1,4,1,smem,g,cps15,ns8" "32,2,12,4,1,tmem,g,cps15"
echo "== Apertif d=16"
$T Apertif 16 "8,16,25,1,1,smem,tm,cps15" "32,4,12,4,1,tmem,g,cps15" "64,2,1,8,1,smem,g,cps15,ns8" "32,2,12,8,1,tmem,g,cps15"
echo "== Apertif d=64"
$T Apertif 64 "8,16,25,1,1,smem,tm,cps15" "32,4,12,8,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps8,occ" "32,2,12,8,1,tmem,g,cps15"
echo "== LOFAR d=2"
$T LOFAR 2 "160,1,5,2,1,smem,cps15" "256,1,4,2,1,smem,g,cps15,ns4"
echo "== LOFAR d=64"
$T LOFAR 64 "160,1,10,4,2,smem,tm,pk"
} > gpurun_out/small_d4.txt 2>&1
{
for L in "" tools/ab/libdedisp_pipe200.so tools/ab/libdedisp_pipe200g2.so tools/ab/libdedisp_lb200.so tools/ab/libdedisp_pipe208.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,12,8,1,tmem,g,cps8"
done
} > gpurun_out/ab4.txt 2>&1
tail -3 gpurun_out/parity4.log
