"""Expert-parallel MoE dispatch / combine over the nimble all-to-allv.

The paper's application context: MoE layers route tokens to
experts that live on other ranks, and a skewed router turns the dispatch into
exactly the skewed all-to-allv this library accelerates.  This module is the
upstream caller: the byte movement is
`Comm.alltoallv` (the sm_100a forwarding engine); PyTorch only does the index
bookkeeping around it (argsort / gather / index_add).  Two faces:
`MoEDispatcher` (registered staging buffers, zero copy, inference) and the
`nimble_b200::alltoallv_rows` custom operator with autograd behind the
differentiable `dispatch` / `combine` functions (training).

Layout: experts are block-distributed, expert e lives on rank e // E_local.
dispatch() sends every (token, k) assignment's hidden vector to its expert's
rank, grouped by destination rank and, within a rank, by (token, k) order;
combine() brings the expert outputs back and reduces them with the router
weights.  Send / receive staging buffers are allocated once at capacity and
registered, so the exchange runs zero copy (receiver-driven pulls where a
port is ingress-bound).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .comm import Comm


@dataclass
class DispatchHandle:
    order: torch.Tensor          # [A] assignment ids (token*k + j) in send order
    send_counts: list            # rows per destination rank
    recv_counts: list            # rows per source rank
    num_tokens: int
    topk: int


class MoEDispatcher:
    """dispatch / combine for `num_experts` experts block-distributed over `comm`."""

    def __init__(self, comm: Comm, num_experts: int, hidden: int, dtype=torch.bfloat16,
                 max_tokens: int = 4096, topk: int = 2):
        if num_experts % comm.nranks:
            raise ValueError("num_experts must be a multiple of the rank count")
        self.comm, self.R, self.hidden, self.dtype = comm, comm.nranks, hidden, dtype
        self.experts_per_rank = num_experts // comm.nranks
        self.elem = torch.tensor([], dtype=dtype).element_size()
        self.row = hidden * self.elem
        cap_send = max_tokens * topk
        cap_recv = max_tokens * topk * comm.nranks      # every rank may route everything here
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send_buf = torch.empty(cap_send, hidden, dtype=dtype, device=dev)
        self.recv_buf = torch.empty(cap_recv, hidden, dtype=dtype, device=dev)
        self.back_buf = torch.empty(cap_send, hidden, dtype=dtype, device=dev)
        self.send_ids = torch.empty(cap_send, dtype=torch.int32, device=dev)
        self.recv_ids = torch.empty(cap_recv, dtype=torch.int32, device=dev)
        self.count_out = torch.zeros(self.R, dtype=torch.int64, device=dev)
        self.count_in = torch.zeros(self.R, dtype=torch.int64, device=dev)
        self._handles = [comm.register(t) for t in (self.send_buf, self.recv_buf, self.back_buf,
                                                    self.send_ids, self.recv_ids)]
        self.cap_send, self.cap_recv = cap_send, cap_recv

    def close(self):
        for h in self._handles:
            self.comm.deregister(h)
        self._handles = []

    @staticmethod
    def _displs(counts):
        out, acc = [], 0
        for c in counts:
            out.append(acc)
            acc += c
        return out

    @staticmethod
    def _enter(stream):
        """Exchanges on `stream` see the current stream's work (buffers filled)."""
        if stream is not None:
            stream.wait_stream(torch.cuda.current_stream())

    @staticmethod
    def _leave(stream):
        """The current stream sees the exchanges' results."""
        if stream is not None:
            torch.cuda.current_stream().wait_stream(stream)

    def dispatch(self, x: torch.Tensor, topk_ids: torch.Tensor, stream=None):
        """x [T, H], topk_ids [T, k] (int) -> (recv_x [N, H], recv_expert [N] local ids, handle).
        `stream` (optional, a torch.cuda.Stream): run the exchanges there; it is
        ordered after the current stream's work and before the current stream's
        later work."""
        T, k = topk_ids.shape
        if T * k > self.cap_send:
            raise ValueError("more assignments than the dispatcher's capacity")
        flat = topk_ids.reshape(-1).to(torch.int64)
        dest = flat // self.experts_per_rank
        order = torch.argsort(dest, stable=True)
        n = T * k
        torch.index_select(x, 0, order // k, out=self.send_buf[:n])
        self.send_ids[:n] = (flat[order] % self.experts_per_rank).to(torch.int32)
        self.count_out.copy_(torch.bincount(dest, minlength=self.R))
        # counts first (one int64 per peer), then the rows
        self._enter(stream)
        self.comm.alltoall(self.count_out, self.count_in, 8, stream)
        # the counts are read on the host next: wait with the GIL released
        # (tolist() would block holding it -- a peer rank's thread in this
        # process could then never launch the exchange this one waits for)
        (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        send_counts = self.count_out.tolist()
        recv_counts = self.count_in.tolist()
        if sum(recv_counts) > self.cap_recv:
            raise ValueError("received more rows than the dispatcher's capacity")
        sb = [c * self.row for c in send_counts]
        rb = [c * self.row for c in recv_counts]
        self.comm.alltoallv(self.send_buf, sb, self._displs(sb), self.recv_buf, rb, self._displs(rb), stream)
        si = [c * 4 for c in send_counts]
        ri = [c * 4 for c in recv_counts]
        self.comm.alltoallv(self.send_ids, si, self._displs(si), self.recv_ids, ri, self._displs(ri), stream)
        self._leave(stream)
        m = sum(recv_counts)
        return self.recv_buf[:m], self.recv_ids[:m], DispatchHandle(order, send_counts, recv_counts, T, k)

    def combine(self, y: torch.Tensor, handle: DispatchHandle, weights: torch.Tensor | None = None, stream=None):
        """y [N, H] expert outputs in dispatch-receive order -> out [T, H] (router-weighted sum)."""
        m = sum(handle.recv_counts)
        if y.data_ptr() != self.recv_buf.data_ptr():
            self.recv_buf[:m].copy_(y)
        sb = [c * self.row for c in handle.recv_counts]
        rb = [c * self.row for c in handle.send_counts]
        self._enter(stream)
        self.comm.alltoallv(self.recv_buf, sb, self._displs(sb), self.back_buf, rb, self._displs(rb), stream)
        self._leave(stream)
        n = handle.num_tokens * handle.topk
        back = self.back_buf[:n]
        if weights is not None:
            w = weights.reshape(-1)[handle.order].to(back.dtype).unsqueeze(1)
            back = back * w
        out = torch.zeros(handle.num_tokens, self.hidden, dtype=self.dtype, device=back.device)
        out.index_add_(0, handle.order // handle.topk, back)
        return out


# ---------------------------------------------------------------- custom op
#
# The same exchange as a PyTorch custom operator with autograd, so a training
# step can differentiate through dispatch / combine: the backward of an
# all-to-allv of rows is the all-to-allv of the row gradients the other way.

_COMMS: dict = {}


def comm_id(comm: Comm) -> int:
    """Integer handle of `comm` for the custom op (custom ops take no Python objects)."""
    _COMMS[id(comm)] = comm
    return id(comm)


def _prefix(counts):
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += c
    return out


@torch.library.custom_op("nimble_b200::alltoallv_rows", mutates_args=())
def alltoallv_rows(x: torch.Tensor, send_counts: list[int], recv_counts: list[int], comm: int) -> torch.Tensor:
    """x [sum(send_counts), ...] rows grouped by destination rank -> [sum(recv_counts), ...]
    grouped by source rank, through the forwarding engine (nimbleAlltoAllv) on the
    current stream."""
    c = _COMMS[comm]
    x = x.contiguous()
    row = x[0].numel() * x.element_size() if x.shape[0] else int(torch.tensor(x.shape[1:]).prod()) * x.element_size()
    out = x.new_empty((sum(recv_counts),) + tuple(x.shape[1:]))
    sb = [n * row for n in send_counts]
    rb = [n * row for n in recv_counts]
    c.alltoallv(x, sb, _prefix(sb), out, rb, _prefix(rb))
    return out


@alltoallv_rows.register_fake
def _alltoallv_rows_fake(x, send_counts, recv_counts, comm):
    return x.new_empty((sum(recv_counts),) + tuple(x.shape[1:]))


def _a2a_setup(ctx, inputs, output):
    _, ctx.send_counts, ctx.recv_counts, ctx.comm = inputs


def _a2a_backward(ctx, grad):
    return alltoallv_rows(grad.contiguous(), ctx.recv_counts, ctx.send_counts, ctx.comm), None, None, None


alltoallv_rows.register_autograd(_a2a_backward, setup_context=_a2a_setup)


def dispatch(comm: Comm, x: torch.Tensor, topk_ids: torch.Tensor, num_experts: int):
    """Differentiable dispatch: x [T, H], topk_ids [T, k] -> (recv_x [N, H], recv_expert [N] local
    ids, handle).  Rows are grouped by destination rank, (token, k) order within."""
    R = comm.nranks
    epr = num_experts // R
    T, k = topk_ids.shape
    flat = topk_ids.reshape(-1).to(torch.int64)
    dest = flat // epr
    order = torch.argsort(dest, stable=True)
    count_out = torch.bincount(dest, minlength=R)
    count_in = torch.empty_like(count_out)
    comm.alltoall(count_out, count_in, 8)
    torch.cuda.current_stream().synchronize()  # GIL released while waiting (see MoEDispatcher.dispatch)
    sc, rc = count_out.tolist(), count_in.tolist()
    cid = comm_id(comm)
    recv_x = alltoallv_rows(x.index_select(0, order // k), sc, rc, cid)
    recv_e = alltoallv_rows((flat[order] % epr).to(torch.int32).unsqueeze(1), sc, rc, cid).squeeze(1)
    return recv_x, recv_e, DispatchHandle(order, sc, rc, T, k)


def combine(comm: Comm, y: torch.Tensor, handle: DispatchHandle, weights: torch.Tensor | None = None):
    """Differentiable combine: y [N, H] in dispatch-receive order -> out [T, H], the
    router-weighted sum over each token's k assignments."""
    back = alltoallv_rows(y, handle.recv_counts, handle.send_counts, comm_id(comm))
    if weights is not None:
        back = back * weights.reshape(-1)[handle.order].to(back.dtype).unsqueeze(1)
    out = torch.zeros(handle.num_tokens, y.shape[1], dtype=y.dtype, device=y.device)
    return out.index_add(0, handle.order // handle.topk, back)


__all__ = ["MoEDispatcher", "DispatchHandle", "alltoallv_rows", "dispatch", "combine", "comm_id", "_lib"]
