mkdir -p gpurun_out/st
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mstep_parity and tc" 2>&1 | tail -15
for c in 3 2 1; do
VMFA_STATS=tc timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/st/c$c.json 2> gpurun_out/st/c$c.err
echo "config $c rc=$?"; tail -2 gpurun_out/st/c$c.err
python -c "
import json; d=json.load(open('gpurun_out/st/c$c.json')); print($c, 'ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
