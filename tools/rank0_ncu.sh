#!/bin/bash
# torchrun --no-python ... bash tools/rank0_ncu.sh OUT.csv SKIP COUNT -- <python args>
# Rank NCU_RANK (default 0) runs under Nsight Compute with a SINGLE-PASS metric set (NVLink
# tx/rx user-data and protocol bytes, DRAM bytes, duration) on the forwarding
# engine's launches; the other ranks run plainly.  One pass means no kernel
# replay, so the multi-rank exchange runs exactly as without the profiler
# (a replayed launch would wait for peers that do not replay: rank 0's wait
# timeout is shortened so that case fails fast instead of hanging).
out=$1; skip=$2; count=$3; shift 3; [ "$1" = "--" ] && shift
if [ "${RANK:-0}" = "${NCU_RANK:-0}" ]; then
  export NIMBLE_PDL=${NIMBLE_PDL:-0}
  export NIMBLE_TIMEOUT_MS=${NIMBLE_TIMEOUT_MS:-5000}
  exec ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes_data_protocol.sum \
    -k regex:exchange_kernel --launch-skip "$skip" --launch-count "$count" --clock-control none --cache-control none \
    --replay-mode kernel --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi
