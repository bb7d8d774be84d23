# round-2 4-GPU session: MoE caller vs NCCL with the round-2 engine; c5 push vs pull (block timing) (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4i
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for T in 512 4096; do
  MOE_T=$T timeout 600 $TR --nproc-per-node 4 --master-port 2970$((T % 7)) tools/moe_bench.py > ${O}_moe_T$T.jsonl 2> ${O}_moe_T$T.err
  echo "moe T=$T: $(grep -c '^{' ${O}_moe_T$T.jsonl) rows"
done
for pl in 0 1; do
  SWEEP_PULL=$pl SWEEP_PUSH_CHUNK=$([ $pl = 1 ] && echo 32768 || echo 0) SWEEP_CASES=c5 timeout 400 $TR --nproc-per-node 4 --master-port 2971$pl tools/sweeps.py > ${O}_c5_pull$pl.jsonl 2> ${O}_c5_pull$pl.err
done
echo done
