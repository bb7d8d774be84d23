# round-2 4-GPU experiment session (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for spec in "c3 256 0" "c3 64 0" "c5 256 0" "c3 256 1"; do
  set -- $spec
  timeout 400 $TR --master-port 2957$4 --no-python env NCU_RANK=$3 bash tools/rank0_ncu.sh ${O}_ncu_$1_$2_r$3.csv 3 3 -- tools/ncu_exchange.py --case $1 --per-rank-mib $2 > ${O}_ncu_$1_$2_r$3.out 2>&1
  echo "ncu $spec rc=$?"
done
TRACE_PULL=0 TRACE_KIB=65536,262144 timeout 300 $TR --master-port 29581 tools/trace_probe.py > ${O}_trace.txt 2>&1
TRACE_PULL=0 TRACE_KIB=65536 TRACE_RATIO=0.333333 timeout 300 $TR --master-port 29582 tools/trace_probe.py > ${O}_trace_c5.txt 2>&1
timeout 300 python tools/ce_probe.py 256 > ${O}_ce256.jsonl 2> ${O}_ce256.err
timeout 300 python tools/ce_probe.py 64 > ${O}_ce64.jsonl 2> ${O}_ce64.err
for pc in 32768 65536; do
  SWEEP_NCCL=0 SWEEP_PULL=1 SWEEP_PUSH_CHUNK=$pc SWEEP_CASES=c5,c3 timeout 400 $TR --master-port 29583 tools/sweeps.py > ${O}_push$pc.jsonl 2> ${O}_push$pc.err
done
NIMBLE_PDL=0 SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3 timeout 300 $TR --master-port 29584 tools/sweeps.py > ${O}_nopdl64.jsonl 2> ${O}_nopdl64.err
echo done
