# pytest -m gpu (optionally a -k selection) + config-3 bench phase split
mkdir -p gpurun_out/q
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15 > gpurun_out/q/pytest.log
tail -3 gpurun_out/q/pytest.log
for c in ${CONFIGS:-3}; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/q/c$c.json 2> gpurun_out/q/c$c.err
echo "config $c rc=$?"; tail -2 gpurun_out/q/c$c.err
python -c "
import json; d=json.load(open('gpurun_out/q/c$c.json')); print('ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
