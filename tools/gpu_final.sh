cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
mkdir -p gpurun_out/tuning_small
timeout 600 python tune.py --setup Apertif --dms 2 --dms 4 --dms 8 --dms 16 --dms 32 --out gpurun_out/tuning_small > $O/tune_small.log 2>&1
tail -6 $O/tune_small.log
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1
tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python bench.py --setup LOFAR --steps 10 --warmup 3 --no-cpu > $O/bench_lofar.json 2> $O/bench_lofar.err
./tools/dropin_bench.bin Apertif 4096 10 > $O/dropin_ap.json 2>&1
./tools/dropin_bench.bin LOFAR 4096 5 > $O/dropin_lofar.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_dropin.csv ./tools/dropin_bench.bin Apertif 4096 2 > $O/ncu_dropin.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tmemwin -s 3 -c 1 -o $O/k5 python tools/time_configs.py Apertif 4096 "32,4,12,8,1,tmem,g,cps15" > $O/ncu_k5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_smem -s 3 -c 1 -o $O/k3_lofar python tools/time_configs.py LOFAR 4096 "160,1,10,4,2,smem,tm,pk" > $O/ncu_k3_lofar.log 2>&1
cat $O/bench.json
