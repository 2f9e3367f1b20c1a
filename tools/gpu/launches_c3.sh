# ncu launch list of the config-3 bench (profile-only: 2 warm-up E-steps,
# W warm-up iterations, 2 iterations), summarised over the last iteration
mkdir -p gpurun_out/prof
VMFA_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --profile-only --warmup ${W:-1} --no-cpu-baseline --no-e2e --no-exact-ll ${BENCH_ARGS:-} > gpurun_out/prof/launches.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/prof/launches.log
python tools/launch_summary.py gpurun_out/prof/launches.csv > gpurun_out/prof/launch_summary_all.txt
head -60 gpurun_out/prof/launch_summary_all.txt
