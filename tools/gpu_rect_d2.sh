# small-d rectangle sweep outside the tuner space (stage count 2..4, boxes of 32..128 channels)
cd $GRAFT_REPO_ROOT
O=gpurun_out/rect_d2
mkdir -p $O
timeout 900 python tools/time_configs.py --cold Apertif 2 $(cat tools/rect_d2_specs.txt) > $O/d2.txt 2>&1
sort -k3 -g $O/d2.txt | grep " ms " | head -15
