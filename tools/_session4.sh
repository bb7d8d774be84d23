# round-2 4-GPU session: split peer signaling A/B + correctness (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4k
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export CUDA_MODULE_LOADING=EAGER
timeout 1200 python -m pytest tests/test_gpu_comm.py -k "proc or thread4" -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest: $(tail -1 ${O}_pytest.txt)"
unset CUDA_MODULE_LOADING
for sp in 1 0; do
  NIMBLE_SPLIT_SIGNAL=$sp SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c3k,c4 timeout 600 $TR --nproc-per-node 4 --master-port 2973$sp tools/sweeps.py > ${O}_split${sp}.jsonl 2> ${O}_split${sp}.err
done
echo done
