cd $GRAFT_REPO_ROOT
T="python tools/time_configs.py --cold"
$T LOFAR 4096 "160,1,10,4,2,smem,tm,pk" "160,2,10,4,1,smem,tm,pk" "160,2,10,4,2,smem,tm,pk" "160,2,20,4,1,smem,tm,pk" "160,1,20,4,2,smem,tm,pk" "160,1,20,4,1,smem,tm,pk" "160,2,10,4,1,smem,tm,pk,ns3"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tuned_configs or packed or large_delay" 2>&1 | tail -2
