# round-2 4-GPU session: per-pair push/pull split on balanced ports (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4m
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for mk in 0 4 10; do
  NIMBLE_PUSH_DISTANCES=$mk SWEEP_NCCL=0 SWEEP_CASES=c5,c3 timeout 500 $TR --nproc-per-node 4 --master-port 29770 tools/sweeps.py > ${O}_mask${mk}.jsonl 2> ${O}_mask${mk}.err
  echo "mask $mk: $(grep -c '^{' ${O}_mask${mk}.jsonl)"
done
echo done
