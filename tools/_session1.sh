# final 1-GPU verification (development aid)
mkdir -p gpurun_out
O=gpurun_out/s1f
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 400 -p no:cacheprovider > ${O}_gputest.txt 2>&1
echo "gputest: $(tail -1 ${O}_gputest.txt)"
timeout 200 python __graft_entry__.py smoke > ${O}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?"
echo done
