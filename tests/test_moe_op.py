"""The MoE exchange as a PyTorch custom operator (CPU: registration, fake
implementation for tracing; the GPU parity + gradient test is in
test_gpu_comm.py::test_moe_custom_op_forward_and_gradients)."""
import pytest

torch = pytest.importorskip("torch")


def test_custom_op_is_registered_with_fake_and_autograd():
    from paper_2604_00317_b200 import moe
    op = torch.ops.nimble_b200.alltoallv_rows
    assert op is not None
    x = torch.empty(7, 5, device="meta")
    y = moe._alltoallv_rows_fake(x, [3, 4], [2, 6], 0)
    assert y.shape == (8, 5) and y.device.type == "meta"
    ctx = type("Ctx", (), {})()
    moe._a2a_setup(ctx, (x, [3, 4], [2, 6], 0), y)
    assert (ctx.send_counts, ctx.recv_counts, ctx.comm) == ([3, 4], [2, 6], 0)
