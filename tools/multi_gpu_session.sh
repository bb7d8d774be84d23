#!/bin/bash
# One multi-GPU measurement session (gpurun --gpus N): proc-mode parity tests,
# bench lines at N (default + fresh matrices), per-call host cost, the
# BASELINE sweeps at 64 MiB and 256 MiB per rank with NVML NVLink counters,
# and a single-pass ncu NVLink / DRAM capture of rank 0's engine launches.
# Everything lands in gpurun_out/mg_<N>_*.
N=${1:-4}
O=gpurun_out/mg_${N}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
python -c "import __graft_entry__ as g; g.build()" > ${O}_build.log 2>&1
nvidia-smi topo -m > ${O}_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_comm.py -k "proc" -q -p no:cacheprovider > ${O}_pytest_proc.txt 2>&1
echo "pytest proc: $(tail -1 ${O}_pytest_proc.txt)"
timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
echo "bench: $(cut -c1-300 ${O}_bench.json)"
timeout 300 $TR bench.py --gpus $N --steps 20 --warmup 5 --fresh-matrix --no-e2e --no-baselines > ${O}_bench_fresh.json 2> ${O}_bench_fresh.err
echo "bench fresh: $(cut -c1-300 ${O}_bench_fresh.json)"
timeout 300 $TR tools/fresh_matrix_probe.py > ${O}_fresh_probe.json 2> ${O}_fresh_probe.err
SWEEP_NVML=1 SWEEP_PER_RANK_MIB=64 SWEEP_CASES=c3,c5 timeout 900 $TR tools/sweeps.py > ${O}_sweep64.jsonl 2> ${O}_sweep64.err
SWEEP_NVML=1 SWEEP_CASES=c3,c3a,c5,c4,c1,c2 timeout 1200 $TR tools/sweeps.py > ${O}_sweep256.jsonl 2> ${O}_sweep256.err
echo "sweeps: $(wc -l < ${O}_sweep64.jsonl) + $(wc -l < ${O}_sweep256.jsonl) rows"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 --no-python \
  bash tools/rank0_ncu.sh ${O}_ncu_nvlink.csv 5 3 -- bench.py --gpus $N --steps 3 --warmup 5 --no-e2e --no-baselines --no-cpu \
  > ${O}_ncu_run.json 2> ${O}_ncu_run.err
echo "ncu rc=$? lines=$(wc -l < ${O}_ncu_nvlink.csv)"
