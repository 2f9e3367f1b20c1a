for i in 1 2 3; do
for d in "" "--dump-state /tmp/two$i"; do
VMFA_SORT_CHECK=${CHK:-0} MASTER_ADDR=127.0.0.1 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2953$i bench.py --config 2 --rows 12000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-exact-ll --backend gloo --gpus 2 $d > gpurun_out/tr$i.log 2>&1; echo "run $i [$d] rc=$?"; grep "VmfaError\|check failed" gpurun_out/tr$i.log | head -3
done; done
