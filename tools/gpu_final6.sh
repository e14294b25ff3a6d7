cd $GRAFT_REPO_ROOT
O=gpurun_out/final6
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1
tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python bench.py --setup LOFAR --steps 10 --warmup 3 --no-cpu > $O/bench_lofar.json 2> $O/bench_lofar.err
./tools/dropin_bench.bin Apertif 4096 10 > $O/dropin_ap.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
cat $O/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
tail -1 $O/bench_reference.json | cut -c1-400
