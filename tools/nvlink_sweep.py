"""Engine-knob sweep over NVLink (development aid; run under torchrun).

Prints, on rank 0, one line per (knob setting, workload) with GB/s and the
fraction of the MCF port bound."""
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
    ctas_list = [int(x) for x in os.environ.get("SWEEP_CTAS", "32,64,96,148").split(",")]
    chunks = [int(x) for x in os.environ.get("SWEEP_CHUNK_KIB", "512").split(",")]
    pulls = [int(x) for x in os.environ.get("SWEEP_PULL", "0").split(",")]
    ratios = [float(x) for x in os.environ.get("SWEEP_RATIOS", "0.7").split(",")]
    for pull in pulls:
        for chunk_kib in chunks:
            for ctas in ctas_list:
                comm.set_config(ctas=ctas, pipe_chunk=chunk_kib * 1024, pull=pull,
                                p2p_buffer=min(64, max(2, 10 * 1024 // chunk_kib)) * chunk_kib * 1024)
                runs = [("p2p256", comm.bench_p2p(256 * MiB, 0, 1, warmup=2, iters=8))]
                for r in ratios:
                    runs.append((f"skew{r:.2f}", comm.bench_skewed(256 * MiB, r, 0, warmup=2, iters=8)))
                if rank == 0:
                    for name, r in runs:
                        print(f"pull={pull} chunk={chunk_kib}K ctas={ctas:3d} {name}: {r['gbps_effective']:8.1f} GB/s "
                              f"t={r['seconds_median']*1e3:.3f}ms bound={r['bound_seconds']*1e3:.3f}ms "
                              f"frac={r['bound_seconds']/r['seconds_median']:.3f} bad={r['mismatches']}", flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
