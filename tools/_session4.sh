# round-2 4-GPU session: direct-chunk sweep for mid sizes (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4h
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SWEEP_NCCL=0 SWEEP_CHUNKS=16384,32768,65536 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3k,c4,c3 timeout 900 $TR --nproc-per-node 4 --master-port 29690 tools/sweeps.py > ${O}_chunks.jsonl 2> ${O}_chunks.err
echo done
