# ncu launch list of the bench's profile-only run (warm-up + 2 steps): kernel
# durations, summarised per kernel name over the last iteration's launches
# (plain launches: ncu fails graph-launched k_score_ws nodes with LaunchFailed)
mkdir -p gpurun_out/prof
VMFA_GRAPH=${VMFA_GRAPH:-0} timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --profile-only --no-cpu-baseline --no-e2e --no-exact-ll ${BENCH_ARGS:-} > gpurun_out/prof/launches.log 2>&1
python tools/launch_summary.py gpurun_out/prof/launches.csv
