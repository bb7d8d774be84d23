# round-2 4-GPU session: relay ring geometry (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4l
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for g in "0 0" "131072 33554432" "262144 67108864"; do
  set -- $g
  if [ "$1" = "0" ]; then E=""; else E="SWEEP_PIPE_CHUNK=$1 SWEEP_P2P_BUFFER=$2"; fi
  env $E SWEEP_NCCL=0 SWEEP_CASES=c1 timeout 400 $TR --nproc-per-node 3 --master-port 29740 tools/sweeps.py > ${O}_c1_$1.jsonl 2> ${O}_c1_$1.err
  env $E SWEEP_NCCL=0 SWEEP_CASES=c2,cal timeout 600 $TR --nproc-per-node 4 --master-port 29741 tools/sweeps.py > ${O}_c2_$1.jsonl 2> ${O}_c2_$1.err
  echo "geometry $1 $2: $(grep -c '^{' ${O}_c1_$1.jsonl) + $(grep -c '^{' ${O}_c2_$1.jsonl) rows"
done
TRACE_CASE=relay TRACE_PULL=0 TRACE_KIB=65536 timeout 300 $TR --nproc-per-node 3 --master-port 29742 tools/trace_probe.py > ${O}_trace_relay.txt 2>&1
echo done
