mkdir -p gpurun_out
rm -f gpurun_out/.ncu_uid_*
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
cat > /tmp/r0c.sh <<EOS
export NCU_DUMP_AFTER_S=45 NIMBLE_PDL=0 NIMBLE_TIMEOUT_MS=20000
if [ "\$RANK" = "0" ]; then exec ncu --metrics gpu__time_duration.sum --replay-mode application -c 40 python tools/ncu_exchange.py --per-rank-mib 64 --calls 4; else exec python tools/ncu_exchange.py --per-rank-mib 64 --calls 4; fi
EOS
cat > /tmp/r0d.sh <<EOS
export NCU_DUMP_AFTER_S=45 NIMBLE_PDL=0 NIMBLE_TIMEOUT_MS=20000
if [ "\$RANK" = "0" ]; then exec ncu --metrics gpu__time_duration.sum -c 40 python tools/ncu_exchange.py --per-rank-mib 64 --calls 4; else exec python tools/ncu_exchange.py --per-rank-mib 64 --calls 4; fi
EOS
timeout 150 $TR --master-port 29593 --no-python bash /tmp/r0d.sh > gpurun_out/ncu2d.out 2>&1; echo "d rc=$?" > gpurun_out/ncu2_rc.txt
rm -f gpurun_out/.ncu_uid_*
timeout 150 $TR --master-port 29594 --no-python bash /tmp/r0c.sh > gpurun_out/ncu2c.out 2>&1; echo "c rc=$?" >> gpurun_out/ncu2_rc.txt
timeout 60 ncu --metrics gpu__time_duration.sum -c 5 python -c "import torch; x=torch.ones(1<<20,device='cuda'); y=x*2; torch.cuda.synchronize(); print('ok')" > gpurun_out/ncu_sanity.txt 2>&1; echo "sanity rc=$?" >> gpurun_out/ncu2_rc.txt
