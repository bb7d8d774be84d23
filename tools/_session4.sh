# round-2 4-GPU session: sweeps with back-to-back timing, chaining A/B, clique ncu attempt (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4d
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for ch in 0 1; do
  NIMBLE_CHAIN=$ch SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c3k,c4 timeout 600 $TR --master-port 2958$ch tools/sweeps.py > ${O}_chain${ch}.jsonl 2> ${O}_chain${ch}.err
done
SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5 timeout 600 $TR --master-port 29587 tools/sweeps.py > ${O}_sweep64.jsonl 2> ${O}_sweep64.err
SWEEP_CASES=c3,c3a,c5,c4,c3k timeout 900 $TR --master-port 29588 tools/sweeps.py > ${O}_sweep256.jsonl 2> ${O}_sweep256.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes_data_protocol.sum"
NIMBLE_TIMEOUT_MS=20000 NIMBLE_PDL=0 timeout 300 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 3 > ${O}_ncu_clique_hot.csv 2> ${O}_ncu_clique_hot.err
echo "ncu clique hot rc=$?"
NIMBLE_TIMEOUT_MS=20000 NIMBLE_PDL=0 timeout 300 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 0 > ${O}_ncu_clique_cold.csv 2> ${O}_ncu_clique_cold.err
echo "ncu clique cold rc=$?"
echo done
