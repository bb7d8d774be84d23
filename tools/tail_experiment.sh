#!/bin/bash
# A/B of the end-of-exchange knobs (schedule.cpp Knobs) on c3 at 64 MiB/rank:
# push span (pushes keyed into [0, a)) and the pull tail cut finer.
N=${1:-4}
O=gpurun_out/tail_${N}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541"
run() {  # tag, env...
  local tag=$1; shift
  env "$@" SWEEP_NCCL=0 SWEEP_PER_RANK_MIB=${PER:-64} SWEEP_CASES=c3 timeout 300 $TR tools/sweeps.py > ${O}_${tag}.jsonl 2> ${O}_${tag}.err
  python - "$tag" ${O}_${tag}.jsonl <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[2]) if l.startswith("{")]
print(sys.argv[1], " ".join(f"{r['ratio']:.1f}:{r['frac_of_bound']:.3f}{'' if r['mismatched_bytes'] == 0 else '!'}" for r in rows))
PY
}
run base
run span75 NIMBLE_PUSH_SPAN=0.75
run span60 NIMBLE_PUSH_SPAN=0.6
run tail1m NIMBLE_PULL_TAIL=1048576
run tail4m NIMBLE_PULL_TAIL=4194304 NIMBLE_PULL_TAIL_CHUNK=16384
run both NIMBLE_PUSH_SPAN=0.75 NIMBLE_PULL_TAIL=1048576
run both2 NIMBLE_PUSH_SPAN=0.6 NIMBLE_PULL_TAIL=4194304
