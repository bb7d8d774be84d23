# final 4-GPU check after the bounds checks (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4p
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_comm.py -k proc -q -p no:cacheprovider > ${O}_pytest_proc.txt 2>&1
echo "pytest proc: $(tail -1 ${O}_pytest_proc.txt)"
SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5,c4 timeout 400 $TR --nproc-per-node 4 --master-port 29795 tools/sweeps.py > ${O}_sweep64.jsonl 2> ${O}_sweep64.err
echo done
