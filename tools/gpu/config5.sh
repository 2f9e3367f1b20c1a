# config 5's per-GPU work of the 8-GPU run (N = 50M / 8 = 6.25M rows, full
# C = 50 000, H = 64) on one B200
mkdir -p gpurun_out/c5
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 2400 python bench.py --config 5 --n 6250000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-exact-ll \
  > gpurun_out/c5/bench.json 2> gpurun_out/c5/bench.err
echo "config 5 rc=$?"
tail -5 gpurun_out/c5/bench.err
head -c 1500 gpurun_out/c5/bench.json
