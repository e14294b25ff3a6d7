# ncu --set full of the small-d tuned kernels (K6 at d=2, K3 at d=64)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_small
mkdir -p $O
A2=$(python tools/spec_of.py tuning/apertif_2.json)
A64=$(python tools/spec_of.py tuning/apertif_64.json)
python tools/time_configs.py --cold Apertif 2 $A2 > $O/t2.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rect -s 3 -c 1 -o $O/rect_d2 python tools/time_configs.py Apertif 2 $A2 > $O/ncu_rect.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_smem -s 3 -c 1 -o $O/smem_d64 python tools/time_configs.py Apertif 64 $A64 > $O/ncu_smem.log 2>&1
cat $O/t2.txt; tail -n 2 $O/ncu_rect.log $O/ncu_smem.log
