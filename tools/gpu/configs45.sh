# configs 4 and a config-5 shard on one B200 (bench.py --config N), bounded
mkdir -p gpurun_out/c45
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/c45/c4.json 2> gpurun_out/c45/c4.err
echo "config 4 rc=$?"; tail -2 gpurun_out/c45/c4.err
python -c "
import json; d=json.load(open('gpurun_out/c45/c4.json')); print('c4 ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()})"
timeout 1200 python bench.py --config 5 --rows 1000000 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/c45/c5.json 2> gpurun_out/c45/c5.err
echo "config 5 rc=$?"; tail -3 gpurun_out/c45/c5.err
python -c "
import json; d=json.load(open('gpurun_out/c45/c5.json')); print('c5 (1M rows) ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()})"
