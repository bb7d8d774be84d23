# round-2 4-GPU experiment session: epoch chaining A/B (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4c
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_comm.py -k "proc" -q -p no:cacheprovider > ${O}_pytest_proc.txt 2>&1
echo "pytest proc: $(tail -1 ${O}_pytest_proc.txt)"
for ch in 1 0; do
  NIMBLE_CHAIN=$ch SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5,c3k,c4 timeout 600 $TR --master-port 2958$ch tools/sweeps.py > ${O}_chain${ch}.jsonl 2> ${O}_chain${ch}.err
  echo "chain $ch: $(grep -c '^{' ${O}_chain${ch}.jsonl) rows"
done
TRACE_PULL=0 TRACE_KIB=65536,1024 timeout 300 $TR --master-port 29585 tools/trace_probe.py > ${O}_trace.txt 2>&1
timeout 300 $TR --master-port 29586 bench.py --gpus 4 --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
echo "bench: $(cut -c1-200 ${O}_bench.json)"
echo done
