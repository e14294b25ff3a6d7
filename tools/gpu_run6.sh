cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python tools/time_configs.py --cold"
{
echo "== Apertif d=2 (unroll4)"
$T Apertif 2 "32,2,5,1,1,smem,tm,cps15" "128,1,1,2,1,smem,g,cps15,ns4" "64,1,2,2,1,smem,g,cps15,ns8" "96,1,1,2,1,smem,g,cps15,ns8" "32,1,1,2,1,smem,g,cps15,ns8" "64,1,1,2,1,smem,g,cps15,ns8" "32,2,2,1,1,smem,g,cps15,ns6" "32,4,1,1,1,smem,g,cps15,ns8"
echo "== Apertif d=4"
$T Apertif 4 "16,4,10,1,1,smem,tm,cps15" "128,1,1,4,1,smem,g,cps15,ns8" "64,1,1,4,1,smem,g,cps15,ns8" "32,1,2,4,1,smem,g,cps15,ns8" "64,2,1,2,1,smem,g,cps15,ns8" "32,4,1,1,1,smem,g,cps15,ns8"
echo "== Apertif d=8"
$T Apertif 8 "8,8,25,1,1,smem,tm,cps15" "64,2,1,4,1,smem,g,cps15,ns8" "64,1,1,8,1,smem,g,cps15,ns8" "32,2,1,4,1,smem,g,cps15,ns8" "32,4,1,2,1,smem,g,cps15,ns8"
} > gpurun_out/small_d6.txt 2>&1
{
for L in "" tools/ab/libdedisp_pipe.so; do
  echo "== lib ${L:-default}"
  DDB_LIB=$L $T Apertif 4096 "32,4,12,8,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps15" "32,8,12,4,1,tmem,g,cps15" "64,4,12,4,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps8,occ"
  DDB_LIB=$L $T Apertif 64 "32,4,12,4,1,tmem,g,cps15" "32,2,12,4,1,tmem,g,cps15"
done
} > gpurun_out/ab6.txt 2>&1
cat gpurun_out/small_d6.txt gpurun_out/ab6.txt
