# ncu --set full of one late launch of each of the smaller config-3 kernels
mkdir -p gpurun_out/prof
VMFA_GRAPH=0 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:^(k_precompute|k_build_records|k_build_images|k_update|k_gupdate|k_select|k_stats_reduce)$" -s ${SKIP:-20} -c ${COUNT:-8} \
  -o gpurun_out/prof/${OUT:-small} \
  python bench.py --profile-only --warmup 1 --no-cpu-baseline --no-e2e --no-exact-ll ${BENCH_ARGS:-} > gpurun_out/prof/${OUT:-small}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof/${OUT:-small}.log
