# ncu --set full of one launch of kernel $1 (regex) in the bench's profile-only run
mkdir -p gpurun_out/prof
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${SKIP:-2} -c 1 -o gpurun_out/prof/$2 \
  python bench.py --profile-only --no-cpu-baseline --no-e2e --no-exact-ll ${BENCH_ARGS:-} > gpurun_out/prof/$2.log 2>&1
echo "ncu rc=$?"
