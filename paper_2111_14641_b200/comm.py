"""Row sharding of the tall dimension and the per-block sketch allreduce.

The reference is single-process (SPEC.md:13 lists distributed RBGS as a
non-goal); the paper anticipates "only one global synchronization between
distributed processors ... per iteration".  Here the n rows
are cut into contiguous shards, one per rank; every sketch Theta @ X is a sum
over rows, so each rank sketches its own rows (the operators are keyed by
GLOBAL row) and one fp64 sum-allreduce completes it.  The small k-, m- and
p-dimensional state (S, P, R, X) is replicated and every rank runs the same
small solves on the same bits, so no broadcast is ever needed.

`Comm` is a thin wrapper over a `torch.distributed` process group (NCCL on
the GPU box, gloo in the CPU tests); with world size 1 every call is a no-op.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class RowShard:
    """Rows [row0, row0 + n_local) of a global n."""

    n: int
    row0: int
    n_local: int

    @staticmethod
    def split(n: int, world: int, rank: int, align: int = 1) -> "RowShard":
        """Contiguous near-equal shards; boundaries are multiples of `align`
        (2048 keeps SRHT tiles whole, 32 keeps rademacher bit words whole)."""
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} / world {world}")
        units = -(-n // align)
        base, extra = divmod(units, world)
        start_u = rank * base + min(rank, extra)
        cnt_u = base + (1 if rank < extra else 0)
        row0 = min(n, start_u * align)
        end = min(n, (start_u + cnt_u) * align)
        return RowShard(n, row0, end - row0)

    @staticmethod
    def whole(n: int) -> "RowShard":
        return RowShard(n, 0, n)


class Comm:
    """Sum-allreduce over the ranks that share the rows of one factorization."""

    def __init__(self, group=None):
        self.group = group
        self.collectives = 0  # collectives issued (one per block in the sweep)
        self._bufs = {}
        if group is None or not torch.distributed.is_available() or not torch.distributed.is_initialized():
            self.world, self.rank = 1, 0
            self.group = None
        else:
            self.world = torch.distributed.get_world_size(group)
            self.rank = torch.distributed.get_rank(group)

    @property
    def active(self) -> bool:
        return self.world > 1

    def allreduce_(self, *tensors):
        """In-place sum of every tensor across ranks, as ONE collective: the
        tensors are packed into a persistent fp64 buffer (grown on demand,
        no per-call allocation), reduced, unpacked."""
        tensors = tuple(t for t in tensors if t is not None and t.numel() > 0)
        if not self.active or not tensors:
            return tensors
        self.collectives += 1
        if len(tensors) == 1 and tensors[0].is_contiguous():
            torch.distributed.all_reduce(tensors[0], group=self.group)
            return tensors
        total = sum(t.numel() for t in tensors)
        dev = tensors[0].device
        buf = self._bufs.get(dev)
        if buf is None or buf.numel() < total:
            buf = torch.empty(max(total, 1 << 16), dtype=torch.float64, device=dev)
            self._bufs[dev] = buf
        flat = buf[:total]
        off = 0
        for t in tensors:
            n = t.numel()
            dst = flat[off:off + n]
            if t.is_contiguous():
                dst.view_as(t).copy_(t)
            else:  # column-major 2-D view: its transpose is contiguous
                dst.view(t.shape[1], t.shape[0]).copy_(t.t())
            off += n
        torch.distributed.all_reduce(flat, group=self.group)
        off = 0
        for t in tensors:
            n = t.numel()
            src = flat[off:off + n]
            if t.is_contiguous():
                t.copy_(src.view_as(t))
            else:
                t.t().copy_(src.view(t.shape[1], t.shape[0]))
            off += n
        return tensors

    def max_scalar(self, value: float) -> float:
        if not self.active:
            return value
        t = torch.tensor([value], dtype=torch.float64,
                         device="cuda" if torch.distributed.get_backend(self.group) == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=self.group)
        return float(t.item())
