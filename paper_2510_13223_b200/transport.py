"""Host-side plumbing of the N>1 data plane: the library's own NCCL wire and the P2P
error flag.

``NcclWire`` moves the bytes of the two-sided transport (hand-off chunks, q, partials;
PAPER.md:237, :239-244 eq. 11) through the C-ABI -- ``bs_exchange`` on a ``bs_comm`` the
library owns -- so torch.distributed only broadcasts the ncclUniqueId.  The protocol
classes (``ring.ShardedDecodeStep``, ``seqshard.SeqShardedStep``) talk to any object with
the same ``exchange(sends, recvs)`` method; the CPU tests inject one over gloo.

``ErrorFlag`` is the timeout flag of the P2P signals (``bs_wait_signal*``): one int32 in
page-locked host memory the device writes with a system-scope store, so the host can
check it after every step without synchronising.

``nvtx`` marks host submission ranges (a decode step, each layer) for nsys / ncu
``--nvtx`` filtering when ``BS_NVTX=1``; a no-op otherwise.
"""
from __future__ import annotations

import contextlib
import os

import torch
import torch.distributed as dist

_NVTX = os.environ.get("BS_NVTX") == "1"


@contextlib.contextmanager
def nvtx(name: str):
    """NVTX range around the enclosed submissions (BS_NVTX=1; graph capture records the
    ranges once, at capture time)."""
    if not _NVTX or not torch.cuda.is_available():
        yield
        return
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


class NcclWire:
    """A ``bs_comm`` over the ranks of ``group`` (rank numbering of the group)."""

    def __init__(self, group=None):
        from . import Comm, nccl_unique_id
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        self.comm = Comm(obj[0], world, rank)
        self.rank, self.world = rank, world

    def exchange(self, sends, recvs, stream=None) -> None:
        """sends / recvs: [(tensor, peer)] raw bytes, one NCCL group on ``stream``
        (default: the current stream)."""
        self.comm.exchange([(t.reshape(-1), p) for t, p in sends],
                           [(t.reshape(-1), p) for t, p in recvs], stream=stream)

    def close(self) -> None:
        self.comm.close()


class ErrorFlag:
    """Timeout flag shared by a step's wait kernels (pinned host int32, device-visible
    through UVA).  ``check()`` reads it without synchronising: a timeout of step k is seen
    by the next ``enqueue`` (which raises) or by an explicit ``check()`` after a
    synchronize."""

    def __init__(self):
        self.host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.ptr = self.host.data_ptr()

    def set(self) -> bool:
        return int(self.host[0]) != 0

    def check(self, what: str = "P2P transport") -> None:
        if self.set():
            raise RuntimeError(f"{what}: a peer signal timed out (its outputs of that step are "
                               "invalid)")

    def clear(self) -> None:
        self.host[0] = 0
