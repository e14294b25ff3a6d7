cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt
./tools/ubench/fadd.bin > gpurun_out/fadd.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py --quick > gpurun_out/racecheck.log 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/synccheck.log 2>&1
tail -3 gpurun_out/gputest.log
