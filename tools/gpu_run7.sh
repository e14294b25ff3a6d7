cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "rect" > gpurun_out/rect_tests.log 2>&1
tail -15 gpurun_out/rect_tests.log
T="python tools/time_configs.py --cold"
{
echo "== Apertif d=2"
$T Apertif 2 "32,2,5,1,1,smem,tm,cps15" "128,1,1,2,1,rect,g" "128,1,1,2,1,rect,g,cps4" "128,1,1,2,1,rect,g,cps2" "64,1,2,2,1,rect,g" "128,1,2,2,1,rect,g" "256,1,1,2,1,rect,g,cps2" "64,1,1,2,1,rect,g,cps4,ns6" "96,1,1,2,1,rect,g,cps4"
echo "== Apertif d=4"
$T Apertif 4 "16,4,10,1,1,smem,tm,cps15" "128,1,1,4,1,rect,g" "64,1,2,4,1,rect,g" "64,2,1,2,1,rect,g" "128,1,1,4,1,rect,g,cps2" "32,4,1,1,1,rect,g"
echo "== Apertif d=8"
$T Apertif 8 "64,2,1,4,1,smem,g,cps15,ns8" "128,1,1,8,1,rect,g" "64,2,1,4,1,rect,g" "32,4,1,2,1,rect,g" "64,1,2,8,1,rect,g" "128,2,1,4,1,rect,g,cps2"
echo "== Apertif d=16"
$T Apertif 16 "8,16,25,1,1,smem,tm,cps15" "64,2,1,8,1,rect,g" "32,4,1,4,1,rect,g" "64,1,2,16,1,rect,g" "128,1,1,16,1,rect,g" "32,8,1,2,1,rect,g"
echo "== Apertif d=32"
$T Apertif 32 "8,8,25,1,1,smem,tm,cps15" "32,4,1,8,1,rect,g" "64,2,1,16,1,rect,g" "32,8,1,4,1,rect,g" "32,2,1,16,1,rect,g"
echo "== Apertif d=64"
$T Apertif 64 "8,16,25,1,1,smem,tm,cps15" "32,4,1,16,1,rect,g" "32,8,1,8,1,rect,g" "16,8,2,8,1,rect,g" "32,4,2,16,1,rect,g"
} > gpurun_out/rect7.txt 2>&1
cat gpurun_out/rect7.txt
