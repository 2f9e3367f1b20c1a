# Round evidence for profiles/r02 (config 3, the bench default): the bench line
# (no profiler), the ncu launch list of the same workload, and --set full
# captures of the scorer launches and the other top kernels. Summarise with
#   python tools/summarize_ncu.py --round r02 --launches gpurun_out/r02/launches.csv \
#     --full gpurun_out/r02/score.ncu-rep --full2 gpurun_out/r02/other.ncu-rep --bench gpurun_out/r02/bench.json
mkdir -p gpurun_out/r02
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err || { tail -5 gpurun_out/r02/bench.err; exit 1; }
VMFA_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches.csv \
  python bench.py --profile-only --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/r02/launches.log 2>&1
echo "launches rc=$?"
VMFA_GRAPH=0 timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:^k_score_ws$" -s 6 -c 3 \
  -o gpurun_out/r02/score python bench.py --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/r02/score.log 2>&1
echo "score rc=$?"
VMFA_GRAPH=0 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:^(k_stats_mma|k_gupdate|k_select|k_precompute|k_build_images|k_update)$" -s 14 -c 8 \
  -o gpurun_out/r02/other python bench.py --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll > gpurun_out/r02/other.log 2>&1
echo "other rc=$?"
head -c 600 gpurun_out/r02/bench.json
