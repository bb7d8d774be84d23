# round-2 4-GPU session: push lane A/B + correctness (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4f
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export CUDA_MODULE_LOADING=EAGER
timeout 1200 python -m pytest tests/test_gpu_comm.py -k "proc or thread4" -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest: $(tail -1 ${O}_pytest.txt)"
for pl in 1 0; do
  NIMBLE_PUSH_LANE=$pl SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5 timeout 400 $TR --nproc-per-node 4 --master-port 2964$pl tools/sweeps.py > ${O}_lane${pl}_64.jsonl 2> ${O}_lane${pl}_64.err
  NIMBLE_PUSH_LANE=$pl SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=256 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 4 --master-port 2965$pl tools/sweeps.py > ${O}_lane${pl}_256.jsonl 2> ${O}_lane${pl}_256.err
  NIMBLE_PUSH_LANE=$pl SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 3 --master-port 2966$pl tools/sweeps.py > ${O}_lane${pl}_64_w3.jsonl 2> ${O}_lane${pl}_64_w3.err
done
TRACE_PULL=0 TRACE_KIB=65536 timeout 300 $TR --nproc-per-node 4 --master-port 29670 tools/trace_probe.py > ${O}_trace.txt 2>&1
echo done
