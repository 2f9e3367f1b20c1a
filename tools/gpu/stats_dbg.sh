mkdir -p gpurun_out/st
for dbg in 0 1 2 3; do
VMFA_STATS_TC_DBG=$dbg VMFA_STATS=tc timeout 600 python bench.py --config ${CFG:-3} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/st/d$dbg.json 2> gpurun_out/st/d$dbg.err
python -c "
import json; d=json.load(open('gpurun_out/st/d$dbg.json')); print('dbg $dbg stats', round(d['phase_ms']['stats'],3))" 2>&1 | tail -1
done
