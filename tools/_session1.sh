# round-2 1-GPU evidence session (development aid)
mkdir -p gpurun_out
O=gpurun_out/s1
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 400 -p no:cacheprovider > ${O}_gputest.txt 2>&1
echo "gputest: $(tail -1 ${O}_gputest.txt)"
timeout 200 python __graft_entry__.py smoke > ${O}_smoke.txt 2>&1; echo "smoke rc=$?"
export CUDA_MODULE_LOADING=EAGER
timeout 600 python tools/fresh_matrix_probe.py --threads 8 --per-rank-mib 256 > ${O}_fresh_r8.json 2> ${O}_fresh_r8.err
echo "fresh r8 rc=$?"
for tool in memcheck racecheck synccheck; do
  for w in local comm1 thread2; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python tools/sanitize_probe.py $w > ${O}_san_${tool}_${w}.txt 2>&1
    echo "sanitizer $tool $w rc=$?"
  done
done
unset CUDA_MODULE_LOADING
timeout 300 python bench.py > ${O}_bench.json 2> ${O}_bench.err
echo "bench rc=$?"
timeout 300 python bench.py --impl reference > ${O}_bench_ref.json 2> ${O}_bench_ref.err
echo "bench ref rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 3 -c 1 -f -o ${O}_exchange_local python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-baselines > ${O}_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-baselines > ${O}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
echo done
