# round-2 4-GPU session: engine CTA count (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4n
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 148 120 96; do
  SWEEP_CTAS=$n SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5 timeout 400 $TR --nproc-per-node 4 --master-port 29780 tools/sweeps.py > ${O}_ctas$n.jsonl 2> ${O}_ctas$n.err
  echo "ctas $n: $(grep -c '^{' ${O}_ctas$n.jsonl)"
done
echo done
