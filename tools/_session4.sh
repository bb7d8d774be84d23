# round-2 4-GPU session: push-span near 1 A/B + clean trace (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4g
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
TRACE_PULL=0 TRACE_KIB=65536,1024 timeout 300 $TR --nproc-per-node 4 --master-port 29680 tools/trace_probe.py > ${O}_trace.txt 2>&1
for sp in 1.0 0.95 0.9; do
  NIMBLE_PUSH_SPAN=$sp SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 4 --master-port 29681 tools/sweeps.py > ${O}_span${sp}_64.jsonl 2> ${O}_span${sp}_64.err
  NIMBLE_PUSH_SPAN=$sp SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=256 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 4 --master-port 29682 tools/sweeps.py > ${O}_span${sp}_256.jsonl 2> ${O}_span${sp}_256.err
done
NIMBLE_PUSH_SPAN=0.95 TRACE_PULL=0 TRACE_KIB=65536 timeout 300 $TR --nproc-per-node 4 --master-port 29683 tools/trace_probe.py > ${O}_trace_span095.txt 2>&1
echo done
