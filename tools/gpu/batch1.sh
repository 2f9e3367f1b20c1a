mkdir -p gpurun_out/b1
timeout 900 python -m pytest tests -m gpu -x -q -k "estep or select or teacher or free" 2>&1 | tail -3
for c in 3 2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/b1/c$c.json 2> gpurun_out/b1/c$c.err
python -c "
import json; d=json.load(open('gpurun_out/b1/c$c.json')); print($c, 'ms', round(d['ms_per_step'],3), d.get('fp64_rescored_per_step'), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
VMFA_STATS=tc timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/b1/c3tc.json 2> gpurun_out/b1/c3tc.err
python -c "
import json; d=json.load(open('gpurun_out/b1/c3tc.json')); print('stats=tc ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
tail -2 gpurun_out/b1/c3tc.err
# launch list, config 3, same warm-up as the bench
VMFA_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b1/launches_c3.csv \
  python bench.py --profile-only --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/b1/launches_c3.log 2>&1
python tools/launch_summary.py gpurun_out/b1/launches_c3.csv 0 | head -25
# full capture of the scorer (one anchor launch) and the stats kernels
VMFA_GRAPH=0 timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:^(k_score_ws|k_stats_mma)$" -s 14 -c 3 -o gpurun_out/b1/score_stats \
  python bench.py --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/b1/ss.log 2>&1
echo "ncu rc=$?"
VMFA_STATS=tc VMFA_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_stats_tc$" -s 2 -c 1 -o gpurun_out/b1/stats_tc \
  python bench.py --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/b1/stc.log 2>&1
echo "ncu rc=$?"
