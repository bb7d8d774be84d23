mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
NIMBLE_LAUNCH_LOG=1 timeout 300 $TR --master-port 29561 --no-python bash tools/rank0_ncu.sh gpurun_out/ncu2.csv 5 3 -- bench.py --gpus 2 --steps 3 --warmup 5 --no-e2e --no-baselines --no-cpu > gpurun_out/ncu2_run.out 2> gpurun_out/ncu2_run.err
echo "ncu rc=$?" > gpurun_out/ncu2_rc.txt
