# round-2 4-GPU session: 128 KiB pull items (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4o
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for mib in 64 256; do
  SWEEP_PIPE_CHUNK=131072 SWEEP_P2P_BUFFER=10485760 SWEEP_CHUNKS=131072 SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=$mib SWEEP_CASES=c3,c5 timeout 400 $TR --nproc-per-node 4 --master-port 29790 tools/sweeps.py > ${O}_pull128k_$mib.jsonl 2> ${O}_pull128k_$mib.err
  echo "$mib: $(grep -c '^{' ${O}_pull128k_$mib.jsonl)"
done
echo done
