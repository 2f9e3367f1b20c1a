# statistics item size A/B at config 3 (VMFA_STATS_ROWS) + statistics parity tests
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q -k "mstep or stats or suffstats" 2>&1 | tail -3
for r in ${ROWS:-2048 1024 1536 2048 1024}; do
VMFA_STATS_ROWS=$r timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/ab/r$r.json 2> gpurun_out/ab/r$r.err
python -c "
import json; d=json.load(open('gpurun_out/ab/r$r.json')); print('rows $r ms', round(d['ms_per_step'],3), 'stats', round(d['phase_ms']['stats'],3))" 2>&1 | tail -1
done
