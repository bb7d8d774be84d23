# final 4-GPU evidence with the final binary (development aid)
mkdir -p gpurun_out
O=gpurun_out/s4z
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  timeout 400 $TR --nproc-per-node $n --master-port 2975$n bench.py --gpus $n --steps 20 --warmup 5 > ${O}_bench_n$n.json 2> ${O}_bench_n$n.err
  echo "bench n$n: $(cut -c1-160 ${O}_bench_n$n.json)"
done
timeout 400 $TR --nproc-per-node 4 --master-port 29760 bench.py --gpus 4 --steps 20 --warmup 5 --fresh-matrix --no-e2e --no-baselines > ${O}_bench_fresh_n4.json 2> ${O}_bench_fresh_n4.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes_data_protocol.sum"
for mib in 256 64; do
  NIMBLE_TIMEOUT_MS=180000 NIMBLE_PDL=0 timeout 400 ncu --metrics $M -k regex:exchange_kernel --launch-skip 7 --launch-count 1 --csv python tools/ncu_clique.py --gpus 4 --groups 2 --hot 3 --per-rank-mib $mib > ${O}_ncu_hot_$mib.csv 2> ${O}_ncu_hot_$mib.err
  echo "ncu hot $mib rc=$?"
done
echo done
