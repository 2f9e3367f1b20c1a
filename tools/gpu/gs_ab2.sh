mkdir -p gpurun_out/ab
for c in ${CONFIGS:-3 2}; do
for gs in 2 1 2 1; do
VMFA_GSTREAM=$gs timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/ab/g${gs}_c$c.json 2> gpurun_out/ab/g${gs}_c$c.err
python -c "
import json; d=json.load(open('gpurun_out/ab/g${gs}_c$c.json')); print('gstream $gs config $c ms', round(d['ms_per_step'],3), 'F', d['F_last'], 'J', d['joints_per_step'])" 2>&1 | tail -1
done; done
