"""Ghost exchange over torch.distributed (the GhostExchanger protocol,
reference ghost_exchange.cpp:300-398, on NCCL/NVLink for CUDA tensors or gloo
for CPU tensors).

The native C++ transport (`NcclExchanger`, nccl_exchange.cu) is what bench.py
uses; this module runs the same protocol from Python so that the multi-rank
logic -- plan order, receive-in-place into the ghost region, compress
accumulation in ascending source-rank order -- is exercised multi-process on
CPU (gloo) as well.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class TorchExchanger:
    """update (start/finish) and compress for one rank.

    plans: dict(send=[(neighbor, owned_slots)], recv=[(neighbor, n_cells)])
    with the reference plan order (ascending neighbour, ascending cells); the
    receive plans concatenated are the ghost region in storage order.
    """

    def __init__(self, n_owned_cells, dofs_per_cell, send, recv, group=None):
        self.nq = dofs_per_cell
        self.n_owned = n_owned_cells
        self.send = [(nb, torch.as_tensor(slots, dtype=torch.long)) for nb, slots in send]
        self.recv = []
        start = n_owned_cells
        for nb, n in recv:
            self.recv.append((nb, start, start + n))
            start += n
        self.group = group
        self._reqs = None
        self._bufs = None

    @classmethod
    def from_operator(cls, op, group=None):
        lay = op.layout()
        b = lay.owned_cell_begin
        send = [(nb, cells.astype("int64") - b) for nb, cells in op.plans("send")]
        recv = [(nb, len(cells)) for nb, cells in op.plans("recv")]
        return cls(lay.n_owned_cells, lay.dofs_per_cell, send, recv, group)

    def _cells(self, v):
        return v.view(-1, self.nq)

    # update_ghost_values = start + finish (ghost_exchange.cpp:300-351)
    def start_update(self, u):
        if self._reqs is not None:
            raise RuntimeError("update_ghost_values: update already in flight")
        cells = self._cells(u)
        self._bufs, self._reqs = [], []
        for nb, slots in self.send:
            buf = cells.index_select(0, slots.to(u.device)).reshape(-1).contiguous()
            self._bufs.append(buf)
            self._reqs.append(dist.isend(buf, nb, group=self.group))
        for nb, a, e in self.recv:
            self._reqs.append(dist.irecv(cells[a:e].reshape(-1), nb, group=self.group))

    def finish_update(self, u):
        if self._reqs is None:
            raise RuntimeError("finish_ghost_update: no update was started on this vector")
        for r in self._reqs:
            r.wait()
        self._reqs, self._bufs = None, None

    # compress (ghost_exchange.cpp:359-398)
    def compress(self, y):
        cells = self._cells(y)
        reqs, incoming = [], []
        for nb, a, e in self.recv:
            reqs.append(dist.isend(cells[a:e].reshape(-1).contiguous(), nb, group=self.group))
        for nb, slots in self.send:
            buf = torch.empty(len(slots) * self.nq, dtype=y.dtype, device=y.device)
            incoming.append((nb, slots, buf))
            reqs.append(dist.irecv(buf, nb, group=self.group))
        for r in reqs:
            r.wait()
        # ascending source rank: plans are sorted by neighbour
        for nb, slots, buf in incoming:
            cells.index_add_(0, slots.to(y.device), buf.view(-1, self.nq))
        cells[self.n_owned:] = 0


def exchange_apply(exchanger, phase1, phase2, u, y):
    """RankOperator::apply with exchange hooks (operators.cpp:217-264):
    start update, inner cells, finish update, ghost-coupled cells, compress."""
    exchanger.start_update(u)
    phase1(u, y)
    exchanger.finish_update(u)
    phase2(u, y)
    exchanger.compress(y)
