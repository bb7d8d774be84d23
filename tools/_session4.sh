# round-2 4-GPU session: tail pull depth A/B (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4j
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for ti in 0 148 296 592; do
  NIMBLE_TAIL_ITEMS=$ti SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5 timeout 400 $TR --nproc-per-node 4 --master-port 29720 tools/sweeps.py > ${O}_tail${ti}_64.jsonl 2> ${O}_tail${ti}_64.err
done
for ti in 0 296; do
  NIMBLE_TAIL_ITEMS=$ti SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=256 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 4 --master-port 29721 tools/sweeps.py > ${O}_tail${ti}_256.jsonl 2> ${O}_tail${ti}_256.err
done
NIMBLE_TAIL_ITEMS=296 TRACE_PULL=0 TRACE_KIB=65536 timeout 300 $TR --nproc-per-node 4 --master-port 29722 tools/trace_probe.py > ${O}_trace296.txt 2>&1
echo done
