# all gpu tests + config bench phase split
mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-3}; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/ab/c$c.json 2> gpurun_out/ab/c$c.err
python -c "
import json; d=json.load(open('gpurun_out/ab/c$c.json')); print('config $c ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})" 2>&1 | tail -1
done
