"""Ghost exchange over torch.distributed (the GhostExchanger protocol,
reference ghost_exchange.cpp:300-398, on NCCL/NVLink for CUDA tensors or gloo
for CPU tensors).

The native C++ transport (`NcclExchanger`, nccl_exchange.cu) is what bench.py
uses; this module runs the same protocol from Python so that the multi-rank
logic -- plan order, whole-cell or two-layer (Hermite-like) plans,
receive-in-place into the ghost region, compress accumulation in ascending
source-rank order -- is exercised multi-process on CPU (gloo) as well.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class TorchExchanger:
    """update (start/finish) and compress for one rank.

    send / recv: [(neighbor, value_index)] in the reference plan order
    (ascending neighbour, cells ascending, dofs ascending per cell); value
    indices address the rank-local vector (slot * k^d + dof). Whole-cell
    receive plans that are contiguous in the ghost region are received in
    place; partial plans (Hermite-like basis: two layers per coupled face)
    through a buffer and an indexed unpack.
    """

    def __init__(self, owned_size, total_size, send, recv, group=None):
        self.owned_size, self.total_size = owned_size, total_size
        self.send = [(nb, torch.as_tensor(ix, dtype=torch.long)) for nb, ix in send]
        self.recv = []
        for nb, ix in recv:
            ix = torch.as_tensor(ix, dtype=torch.long)
            contiguous = len(ix) > 0 and bool(
                torch.equal(ix, torch.arange(int(ix[0]), int(ix[0]) + len(ix))))
            self.recv.append((nb, ix, contiguous))
        self.group = group
        self._reqs = None
        self._bufs = None

    @classmethod
    def from_operator(cls, op, group=None):
        lay = op.layout()
        return cls(lay.owned_size, lay.total_size, op.plan_values("send"),
                   op.plan_values("recv"), group)

    # update_ghost_values = start + finish (ghost_exchange.cpp:300-351)
    def start_update(self, u):
        if self._reqs is not None:
            raise RuntimeError("update_ghost_values: update already in flight")
        self._bufs, self._reqs, self._unpack = [], [], []
        for nb, ix in self.send:
            buf = u.index_select(0, ix.to(u.device)).contiguous()
            self._bufs.append(buf)
            self._reqs.append(dist.isend(buf, nb, group=self.group))
        for nb, ix, contiguous in self.recv:
            if contiguous:
                a = int(ix[0])
                self._reqs.append(dist.irecv(u[a:a + len(ix)], nb, group=self.group))
            else:
                buf = torch.empty(len(ix), dtype=u.dtype, device=u.device)
                self._unpack.append((ix, buf))
                self._reqs.append(dist.irecv(buf, nb, group=self.group))

    def finish_update(self, u):
        if self._reqs is None:
            raise RuntimeError("finish_ghost_update: no update was started on this vector")
        for r in self._reqs:
            r.wait()
        for ix, buf in self._unpack:
            u.index_copy_(0, ix.to(u.device), buf)
        self._reqs, self._bufs, self._unpack = None, None, None

    # compress (ghost_exchange.cpp:359-398)
    def compress(self, y):
        reqs, incoming = [], []
        for nb, ix, _ in self.recv:
            reqs.append(dist.isend(y.index_select(0, ix.to(y.device)).contiguous(), nb,
                                   group=self.group))
        for nb, ix in self.send:
            buf = torch.empty(len(ix), dtype=y.dtype, device=y.device)
            incoming.append((ix, buf))
            reqs.append(dist.irecv(buf, nb, group=self.group))
        for r in reqs:
            r.wait()
        # ascending source rank: plans are sorted by neighbour
        for ix, buf in incoming:
            y.index_add_(0, ix.to(y.device), buf)
        y[self.owned_size:] = 0


def exchange_apply(exchanger, phase1, phase2, u, y):
    """RankOperator::apply with exchange hooks (operators.cpp:217-264):
    start update, inner cells, finish update, ghost-coupled cells, compress."""
    exchanger.start_update(u)
    phase1(u, y)
    exchanger.finish_update(u)
    phase2(u, y)
    exchanger.compress(y)
