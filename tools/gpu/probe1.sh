mkdir -p gpurun_out/p1
./tools/micro/mma_sync_tput > gpurun_out/p1/mma_sync.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1/c3_launches.csv \
  python bench.py --config 3 --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/p1/c3_ncu.log 2>&1
echo "ncu rc=$?"
timeout 900 python bench.py --config 5 --n 2000000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll \
  > gpurun_out/p1/c5.json 2> gpurun_out/p1/c5.err; echo "config 5 rc=$?"
cat gpurun_out/p1/mma_sync.txt; tail -3 gpurun_out/p1/c5.err; head -c 400 gpurun_out/p1/c5.json
