"""The chunk scheduler's exact output is pinned: 510 per-rank item lists
(skewed / uniform / irregular matrices on 2-8 ranks, both fabric models,
registered / staged / pull receive modes, default and 8 KiB push cuts), hashed.
The item ORDER carries the engine's deadlock-freedom argument (every wait
points at a smaller key), so a change here must be deliberate: regenerate
tests/golden/schedule_hashes.json with NIMBLE_REGEN_SCHEDULE_HASHES=1.
The hashes were produced by the sort-based scheduler; the merge-based one
reproduces them exactly."""
import hashlib
import json
import os

import pytest

from paper_2604_00317_b200 import planner as P

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "schedule_hashes.json")
MiB = 1 << 20


def _hashes(device=False):
    out = {}
    cases = []
    for R in (2, 3, 4, 8):
        for r in (0.0, 0.3, 0.7, 1.0 / (R - 1)):
            cases.append(("skew", R, r, P.gen_skewed_a2av(R, 24 * MiB + 77, r, 0)))
        cases.append(("irr", R, 0, P.gen_irregular(R, 40 * MiB + 5, 0.6, 7)))
    for name, R, r, m in cases:
        for fab in (P.NVSWITCH, P.ALLTOALL):
            topo = P.build_canonical(1, R, 0, 900e9, 0, fab)
            for rank in range(R):
                for staged, pull, pc in ((0, 0, 0), (0b0110, 0b1001, 8192), ((1 << R) - 1, 0, 8192)):
                    items = P.debug_schedule(topo, R, R, m, rank, staged_mask=staged, pull_mask=pull, push_chunk=pc,
                                             device=device)
                    key = f"{name}-{R}-{r:.3f}-{fab}-{rank}-{staged}-{pull}-{pc}"
                    out[key] = hashlib.sha1(json.dumps(items).encode()).hexdigest()
    return out


def test_schedules_match_pinned_hashes(lib):
    got = _hashes()
    if os.environ.get("NIMBLE_REGEN_SCHEDULE_HASHES"):
        with open(GOLDEN, "w") as f:
            json.dump(got, f, indent=0, sort_keys=True)
    with open(GOLDEN) as f:
        want = json.load(f)
    assert set(got) == set(want)
    diff = [k for k in want if got[k] != want[k]]
    assert not diff, f"{len(diff)} schedules changed, e.g. {diff[:3]}"


@pytest.mark.gpu
def test_device_generator_reproduces_pinned_schedules(lib):
    """The GPU merge (engine.cu gen_items_kernel), which schedules every new
    matrix of a communicator, emits the same 510 item lists as the host merge."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with open(GOLDEN) as f:
        want = json.load(f)
    got = _hashes(device=True)
    diff = [k for k in want if got[k] != want[k]]
    assert not diff, f"{len(diff)} schedules differ from the host merge, e.g. {diff[:3]}"
