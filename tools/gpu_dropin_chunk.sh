# drop-in path with DM-chunked execution + overlapped download: tests + timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/dropin_chunk
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py -m gpu -q -x -k "dropin or tuned or drop" > $O/gputest.log 2>&1
tail -3 $O/gputest.log
for rep in 1 2; do
./tools/dropin_bench.bin Apertif 4096 10
./tools/dropin_bench.bin LOFAR 4096 5
./tools/dropin_bench.bin Apertif 64 20
done > $O/dropin.txt 2>&1
cut -c150-420 $O/dropin.txt
