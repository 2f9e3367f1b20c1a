# config-5 shard E-steps (6.25 M rows = 50 M / 8, C = 50 000, H = 64) on one B200
mkdir -p gpurun_out/c5
nvidia-smi --query-gpu=memory.total --format=csv
timeout 1500 python tools/time_estep.py 5 ${ROWS:-6250000} > gpurun_out/c5/estep.log 2>&1
echo "rc=$?"; tail -12 gpurun_out/c5/estep.log
