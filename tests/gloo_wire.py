"""A wire for the multi-process CPU tests (test infrastructure): the byte exchange of the
N>1 protocols (``exchange(sends, recvs)``, the interface of
paper_2510_13223_b200.transport.NcclWire) over torch.distributed gloo, so the CPU tests
run the same protocol code the GPUs run through the library's own NCCL communicator."""
import torch
import torch.distributed as dist


class GlooWire:
    def __init__(self, group=None):
        self.group = group

    def exchange(self, sends, recvs):
        ops = [dist.P2POp(dist.isend, t.reshape(-1).view(torch.uint8), p, group=self.group)
               for t, p in sends]
        ops += [dist.P2POp(dist.irecv, t.reshape(-1).view(torch.uint8), p, group=self.group)
                for t, p in recvs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
