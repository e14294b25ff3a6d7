# Apertif d=2: wider K6 boxes (96..240 channels), 2-3 stages
cd $GRAFT_REPO_ROOT
O=gpurun_out/rect_d2
mkdir -p $O
for rep in 1 2; do
timeout 600 python tools/time_configs.py --cold Apertif 2 $(cat tools/rect_d2_specs2.txt)
done > $O/d2b.txt 2>&1
grep " ms " $O/d2b.txt | sort -k3 -g | head -20
