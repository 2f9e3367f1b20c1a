# One GPU call: tests, smoke, the default bench line (config 3) and the
# reference arm, each bounded by its own timeout. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m "gpu ${PYTEST_SEL:-}" -x -q ${PYTEST_ARGS:-} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; head -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err; head -c 1200 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
