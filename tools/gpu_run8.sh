cd $GRAFT_REPO_ROOT
for a in "a" "a 2" "b 2" "c"; do echo "== $a"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/rect_dbg.py $a 2>&1 | tail -4; done
