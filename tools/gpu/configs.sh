# bench lines for every BASELINE config that fits one B200 (config 5 on a row subset)
mkdir -p gpurun_out/cfg
for c in 1 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll \
    > gpurun_out/cfg/c$c.json 2> gpurun_out/cfg/c$c.err; echo "config $c rc=$?"
done
timeout 900 python bench.py --config 5 --n 200000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-exact-ll \
  > gpurun_out/cfg/c5.json 2> gpurun_out/cfg/c5.err; echo "config 5 rc=$?"
for f in gpurun_out/cfg/*.json; do echo $f; head -c 300 $f; echo; done
tail -5 gpurun_out/cfg/*.err
