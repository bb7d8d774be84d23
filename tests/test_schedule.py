"""The chunk scheduler (csrc/schedule.cpp) on CPU, through nimbleDebugSchedule.

Pins the byte-range convention of SURVEY.md sec. 8(a) row 10 (flows of a pair
take consecutive ranges of its segment in candidate order; ring traffic is cut
into pipe_chunk units with a short tail, pipeline.cpp:85-91) and the ordering
the engine's deadlock-freedom argument relies on (hop 1 of a chunk precedes
hop 2, chunks of a ring in sequence order, on every rank).
"""
import random

import pytest

from paper_2604_00317_b200 import planner as P

MiB, KiB = P.MiB, P.KiB


def _ranges(items):
    return sorted((it["dst"] if it["kind"] != "pull" else it["src"], it["bytes"]) for it in items)


def _contiguous(ranges, start, total):
    pos = start
    for off, n in ranges:
        assert off == pos, (off, pos)
        pos += n
    assert pos == start + total


def _check(topo, R, m, pipe_chunk=64 * KiB, dchunk=64 * KiB, staged=0, pull=0, pchunk=0):
    plan = P.plan(topo, R, R, m)
    sched = {r: P.debug_schedule(topo, R, R, m, r, pipe_chunk=pipe_chunk, direct_chunk=dchunk,
                                 staged_mask=staged, pull_mask=pull, push_chunk=pchunk) for r in range(R)}
    for pp in plan.pairs:
        s, d = pp.src, pp.dst
        off = 0
        for cand, nbytes in pp.flows:
            c = pp.candidates[cand]
            nbytes = int(nbytes)
            if c.cls == "direct":
                push = [it for it in sched[s] if it["kind"] == "push" and it["peer"] == d]
                assert all(it["bytes"] <= (pchunk or dchunk) for it in push)
                _contiguous(_ranges(push), off, nbytes)
                assert [it["seq"] for it in push] == list(range(len(push)))
                if (pull >> s) & 1:
                    pl = [it for it in sched[d] if it["kind"] == "pull" and it["peer"] == s]
                    _contiguous(_ranges(pl), off, nbytes)
                    assert all(it["bytes"] <= dchunk for it in pl)
                if (staged >> s) & 1:  # drained through d's self ring, same chunking
                    fw = [it for it in sched[d] if it["kind"] == "forward" and it["aux"] == s and it["peer"] == d]
                    assert [(it["dst"], it["bytes"], it["seq"]) for it in fw] == \
                           [(it["dst"], it["bytes"], it["seq"]) for it in push]
            else:
                v = c.via
                st = [it for it in sched[s] if it["kind"] == "stage" and it["peer"] == v and it["aux"] == d]
                fw = [it for it in sched[v] if it["kind"] == "forward" and it["aux"] == s and it["peer"] == d]
                _contiguous(_ranges(st), off, nbytes)
                assert all(it["bytes"] == pipe_chunk for it in st[:-1]) and 0 < st[-1]["bytes"] <= pipe_chunk
                assert [it["seq"] for it in st] == list(range(len(st)))  # ring order on the stager
                assert [(it["dst"], it["bytes"], it["seq"]) for it in fw] == \
                       [(it["dst"], it["bytes"], it["seq"]) for it in st]  # same chunks, same order on the relay
            off += nbytes
        assert off == pp.demand
    return plan, sched


def test_nvswitch_skewed_direct_only(lib):
    t = P.build_canonical(1, 8, 0, 900e9, 0, P.NVSWITCH)
    m = P.gen_skewed_a2av(8, 37 * MiB + 5, 0.7, 0)
    plan, sched = _check(t, 8, m)
    assert all(it["kind"] == "push" for r in sched for it in sched[r])


@pytest.mark.parametrize("pchunk", [0, 8 * KiB])
@pytest.mark.parametrize("staged,pull", [(0, 0), (0b1111, 0), (0, 0b1111), (0b0101, 0b1010)])
def test_receive_modes(lib, staged, pull, pchunk):
    t = P.build_canonical(1, 4, 0, 900e9, 0, P.NVSWITCH)
    _check(t, 4, P.gen_irregular(4, 40 * MiB + 77, 0.8, 3), staged=staged, pull=pull, pchunk=pchunk)


def test_mesh_relays_p2p_1gib(lib):  # c2: 0 -> 1 over direct + via 2 + via 3
    t = P.build_canonical(1, 4, 0, 900e9, 0, P.ALLTOALL)
    plan, sched = _check(t, 4, P.gen_p2p(4, 0, 1, 1 << 30))
    assert [int(b) for _, b in plan.pairs[0].flows] == [360710144, 356515840, 356515840]
    assert sum(1 for it in sched[2] if it["kind"] == "forward") == 356515840 // (64 * KiB)


def test_mesh_relays_random(lib):
    rng = random.Random(5)
    for _ in range(6):
        R = rng.randint(3, 6)
        t = P.build_canonical(1, R, 0, 900e9, 0, P.ALLTOALL)
        m = P.gen_skewed_a2av(R, rng.randint(64, 200) * MiB + rng.randint(0, 999), rng.uniform(0.5, 1.0), 0)
        _check(t, R, m, pipe_chunk=rng.choice([64 * KiB, 512 * KiB]))


def test_order_hop1_before_hop2_is_global(lib):
    """Every rank lists ring chunks in sequence order, and interleaves flows by
    progress fraction: the first item of every flow comes before the last item
    of any flow (no flow is starved to the end of the list)."""
    t = P.build_canonical(1, 4, 0, 900e9, 0, P.ALLTOALL)
    m = P.gen_skewed_a2av(4, 256 * MiB, 0.8, 0)
    plan, sched = _check(t, 4, m)
    for r, items in sched.items():
        if not items:
            continue
        firsts, lasts = {}, {}
        for i, it in enumerate(items):
            key = (it["kind"], it["peer"], it["aux"])
            firsts.setdefault(key, i)
            lasts[key] = i
        assert max(firsts.values()) < min(lasts.values()) or len(firsts) == 1
