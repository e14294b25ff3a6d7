cd $GRAFT_REPO_ROOT
for a in "64 32,8,1,2" "32 32,4,1,4" "64 32,16,1,4" "16 32,2,1,4" "64 32,4,1,4 4" "64 32,4,1,4" "16 32,4,1,4" "64 32,8,1,4" "64 32,2,1,8"; do echo "== $a"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/rect_dbg.py $a 2>&1 | grep -E "full|channels|Error" | tail -2; done
