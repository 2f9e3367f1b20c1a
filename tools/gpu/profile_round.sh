# Round evidence for profiles/<round>/ (see profiles/README.md): the bench line
# (no profiler), the ncu launch list of the same command, and one --set full
# capture of the top kernels. Run under gpurun; summarise with
#   python tools/summarize_ncu.py --round r01 --launches gpurun_out/prof/launches.csv \
#       --full gpurun_out/prof/full.ncu-rep --bench gpurun_out/prof/bench.json
mkdir -p gpurun_out/prof
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --profile-only --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/prof/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:^(k_score_ws|k_stats_mma|k_gupdate|k_select)$" -s 12 -c 6 -o gpurun_out/prof/full \
  python bench.py --profile-only --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/prof/full.log 2>&1
echo "profile rc=$?"
