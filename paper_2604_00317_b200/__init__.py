"""nimble-b200: NIMBLE's skew-aware all-to-allv / p2p data path on B200s.

Everything runs through the C ABI of the in-tree libnimble_b200.so
(include/nimble.h); importing a submodule loads it and fails loudly if it is
missing -- there is no CPU fallback.

    planner  -- the reference's planning API (topology, traffic matrices, the
                MCF planner, plan.json), bit-exact with the CPU reference
    comm     -- the NCCL-shaped communicator: init, registration, alltoallv,
                send/recv groups, bench entry points
    moe      -- MoE dispatch / combine over the communicator
"""
