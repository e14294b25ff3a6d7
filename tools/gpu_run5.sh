cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/ubench/tmem_bw.bin > gpurun_out/tmem_bw.txt 2>&1
cat gpurun_out/tmem_bw.txt
