cd $GRAFT_REPO_ROOT
O=gpurun_out/final3
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1
tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python bench.py --setup LOFAR --steps 10 --warmup 3 --no-cpu > $O/bench_lofar.json 2> $O/bench_lofar.err
./tools/dropin_bench.bin Apertif 4096 10 > $O/dropin_ap.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
CFG=$(python -c "
import json;d=json.load(open('tuning/apertif_4096.json'));r=d['records'][d['best_index']];b=r['b200']
f=b['flags'];x=['g'] if f&1 else []
cps=(f>>8)&15; x+=['cps%d'%cps] if cps else []; x+=['wide'] if f&0x20 else []; ns=(f>>12)&15; x+=['ns%d'%ns] if ns else []
print(','.join(map(str,[r['items_time'],r['items_dm'],r['work_time'],r['work_dm'],b['dm_tile_depth'],b['staging']]+x)))")
echo "ncu config: $CFG"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tmemwin -s 3 -c 1 -o $O/k5 python tools/time_configs.py Apertif 4096 "$CFG" > $O/ncu_k5.log 2>&1
cat $O/bench.json
