# round-2 4-GPU session: early posts, pull depth, W=2/3, ncu cold rank, bench lines (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4e
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_comm.py -k "proc" -q -p no:cacheprovider > ${O}_pytest_proc.txt 2>&1
echo "pytest proc: $(tail -1 ${O}_pytest_proc.txt)"
SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c3k,c4 timeout 600 $TR --nproc-per-node 4 --master-port 29591 tools/sweeps.py > ${O}_early64.jsonl 2> ${O}_early64.err
for d in 2 6; do
  NIMBLE_PULL_DEPTH=$d SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3 timeout 400 $TR --nproc-per-node 4 --master-port 2959$d tools/sweeps.py > ${O}_depth$d.jsonl 2> ${O}_depth$d.err
done
for w in 2 3; do
  SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5,c1 timeout 600 $TR --nproc-per-node $w --master-port 2960$w tools/sweeps.py > ${O}_sweep64_w$w.jsonl 2> ${O}_sweep64_w$w.err
  SWEEP_CASES=c3,c5,c4,c1 timeout 900 $TR --nproc-per-node $w --master-port 2961$w tools/sweeps.py > ${O}_sweep256_w$w.jsonl 2> ${O}_sweep256_w$w.err
done
SWEEP_CASES=c2,cal timeout 600 $TR --nproc-per-node 4 --master-port 29620 tools/sweeps.py > ${O}_c2cal.jsonl 2> ${O}_c2cal.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes_data_protocol.sum"
NIMBLE_TIMEOUT_MS=180000 NIMBLE_PDL=0 timeout 400 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 0 > ${O}_ncu_clique_cold.csv 2> ${O}_ncu_clique_cold.err
echo "ncu cold rc=$?"
NIMBLE_TIMEOUT_MS=180000 NIMBLE_PDL=0 timeout 400 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 3 --per-rank-mib 64 > ${O}_ncu_clique_hot64.csv 2> ${O}_ncu_clique_hot64.err
echo "ncu hot64 rc=$?"
NIMBLE_TIMEOUT_MS=180000 NIMBLE_PDL=0 timeout 400 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 3 --ratio 0.333333 > ${O}_ncu_clique_c5.csv 2> ${O}_ncu_clique_c5.err
echo "ncu c5 rc=$?"
for n in 2 4; do
  timeout 400 $TR --nproc-per-node $n --master-port 2963$n bench.py --gpus $n --steps 20 --warmup 5 > ${O}_bench_n$n.json 2> ${O}_bench_n$n.err
  echo "bench n$n: $(cut -c1-160 ${O}_bench_n$n.json)"
done
echo done
