"""Fixed overhead vs asymptotic bandwidth (development aid; torchrun)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00317_b200 import comm as C  # noqa: E402

MiB = 1 << 20


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    uid = [C.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    comm = C.Comm.init_rank(world, uid[0], rank)
    for pull in [int(x) for x in os.environ.get("SWEEP_PULL", "2").split(",")]:
      for dck in [int(x) for x in os.environ.get("SWEEP_DCHUNK_KIB", "64").split(",")]:
       for ctas in [int(x) for x in os.environ.get("SWEEP_CTAS", "0").split(",")]:
        comm.set_config(pull=pull, direct_chunk=dck * 1024, ctas=ctas)
        for ratio in [float(x) for x in os.environ.get("SWEEP_RATIOS", "0.7").split(",")]:
            for mib in [int(x) for x in os.environ.get("SWEEP_MIB", "1,16,64,256,1024").split(",")]:
                r = comm.bench_skewed(mib * MiB, ratio, 0, warmup=3, iters=10)
                if rank == 0:
                    print(f"pull={pull} dchunk={dck}K ctas={ctas} r={ratio:.3f} {mib:5d}MiB: t={r['seconds_median']*1e6:9.1f}us "
                          f"bound={r['bound_seconds']*1e6:9.1f}us frac={r['bound_seconds']/r['seconds_median']:.3f} "
                          f"{r['gbps_effective']:8.1f}GB/s bad={r['mismatches']}", flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
