cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python tools/time_configs.py --cold"
{
echo "== Apertif d=2"
$T Apertif 2 "32,2,5,1,1,smem,tm,cps15" "128,1,1,2,1,smem,g,cps15,ns4" "128,1,1,2,1,smem,g,cps15,ns8" "256,1,1,2,1,smem,g,cps15,ns6" "64,1,2,2,1,smem,g,cps15,ns8" "128,1,2,2,1,smem,g,cps15,ns8" "256,1,2,2,1,smem,g,cps15,ns4" "96,1,1,2,1,smem,g,cps15,ns8" "160,1,1,2,1,smem,cps15,ns8"
echo "== Apertif d=4"
$T Apertif 4 "16,4,10,1,1,smem,tm,cps15" "128,1,1,4,1,smem,g,cps15,ns8" "128,1,2,4,1,smem,g,cps15,ns6" "64,1,2,4,1,smem,g,cps15,ns8" "256,1,1,4,1,smem,g,cps15,ns4" "128,2,1,2,1,smem,g,cps15,ns8"
echo "== Apertif d=8"
$T Apertif 8 "8,8,25,1,1,smem,tm,cps15" "128,1,1,8,1,smem,g,cps15,ns8" "64,1,2,8,1,smem,g,cps15,ns8" "128,2,1,4,1,smem,g,cps15,ns8" "256,1,1,8,1,smem,g,cps15,ns4" "32,2,12,4,1,tmem,g,cps15" "32,1,12,8,1,tmem,g,cps15" "64,1,12,8,1,tmem,g,cps15"
echo "== Apertif d=16"
$T Apertif 16 "8,16,25,1,1,smem,tm,cps15" "32,2,12,8,1,tmem,g,cps15" "32,1,12,8,1,tmem,g,cps15" "64,1,12,8,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps15" "128,1,1,16,1,smem,g,cps15,ns6" "64,2,1,8,1,smem,g,cps15,ns8"
echo "== Apertif d=32"
$T Apertif 32 "8,8,25,1,1,smem,tm,cps15" "32,4,12,8,1,tmem,g,cps15" "32,2,12,8,1,tmem,g,cps15" "32,1,12,8,1,tmem,g,cps15" "64,1,12,8,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps8,occ"
echo "== Apertif d=64"
$T Apertif 64 "8,16,25,1,1,smem,tm,cps15" "32,4,12,8,1,tmem,g,cps15" "32,2,12,8,1,tmem,g,cps15" "32,1,12,8,1,tmem,g,cps15" "64,1,12,8,1,tmem,g,cps15" "32,4,12,4,1,tmem,g,cps8,occ" "32,2,12,4,1,tmem,g,cps15"
echo "== LOFAR d=2"
$T LOFAR 2 "160,1,5,2,1,smem,cps15" "128,1,2,2,1,smem,g,cps15,ns8" "256,1,2,2,1,smem,g,cps15,ns6" "256,1,4,2,1,smem,g,cps15,ns4"
echo "== LOFAR d=8"
$T LOFAR 8 "64,4,25,1,1,smem,tm,cps15" "128,1,2,8,1,smem,g,cps15,ns8" "256,1,1,8,1,smem,g,cps15,ns6"
} > gpurun_out/small_d.txt 2>&1
tail -5 gpurun_out/small_d.txt
timeout 900 python -m pytest tests/test_gpu_checked.py -q > gpurun_out/checked.log 2>&1
tail -2 gpurun_out/checked.log
