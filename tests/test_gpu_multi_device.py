"""The N>1 paths across DISTINCT GPUs -- rank r on cuda:r -- collected with -m gpu and run
whenever at least 2 (or 4) GPUs are visible; skipped cleanly otherwise (gpurun and the
round-end GPU tier offer one GPU; the same-GPU multi-process variants in
test_gpu_ring_p2p.py / test_gpu_seqshard_p2p.py run there).  What only distinct devices
exercise: peer mappings between two GPUs (cudaIpcMemLazyEnablePeerAccess), system-scope
arrival counters and release / acquire flags over NVLink in the fused exchange
("E^(1) ... O^(1) is sent back"), the P2P push of hand-off chunks into a
peer GPU's pool, and the library's own NCCL communicator (bs_exchange, bs_kv_send_layer /
bs_kv_recv_layer) between ranks (eq. 11).  Every case checks against the
oracle: hand-off bytes exact, attention within 2e-2 / 1e-4 (lse)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
import test_gpu_ring_p2p as ring_t
import test_gpu_seqshard_p2p as seq_t

pytestmark = pytest.mark.gpu


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _need(n):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs (rank r on cuda:r); {_gpus()} visible")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(target, world, args_of):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=args_of(r, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not alive, "ranks hung"
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
@pytest.mark.parametrize("fused", [True, False], ids=["fused-exchange", "push-partials"])
@pytest.mark.parametrize("world", [2, 4])
def test_ring_p2p_distinct_gpus(world, fused, graph):
    """The home/cold ring over CUDA IPC between distinct GPUs: q / K/V pushes, hand-off
    chunks pushed into the predecessor's pool, partials stored into (or pushed to) the home
    GPU, last-arriver merges with system-scope atomics; eager and CUDA-graph replay."""
    _need(world)
    _run(ring_t.run_rank, world,
         lambda r, port, errq: (r, world, port, errq, fused, graph, True, "p2p"))


@pytest.mark.parametrize("world", [2, 3])
def test_ring_nccl_distinct_gpus(world):
    """The ring's NCCL transport with the real kernels: q, the token K/V, partials and the
    hand-off (gather -> bs_exchange -> scatter) on the library's own communicators."""
    _need(world)
    _run(ring_t.run_rank, world,
         lambda r, port, errq: (r, world, port, errq, False, False, True, "nccl"))


@pytest.mark.parametrize("world", [2, 4])
def test_seqshard_p2p_distinct_gpus(world):
    _need(world)
    _run(seq_t.run_rank, world, lambda r, port, errq: ("toy", r, world, port, errq, True, "p2p"))


@pytest.mark.parametrize("world", [2, 4])
def test_seqshard_collective_nccl_distinct_gpus(world):
    """The W-way split's two-sided transport: every home's q to every peer and each
    partial to its home through bs_exchange (one NCCL group per exchange)."""
    _need(world)
    _run(seq_t.run_rank, world,
         lambda r, port, errq: ("toy", r, world, port, errq, True, "collective"))


def test_seqshard_c3_shape_4way_distinct_gpus():
    _need(4)
    _run(seq_t.run_rank, 4, lambda r, port, errq: ("c3", r, 4, port, errq, True, "p2p"))


def _sendrecv_rank(rank, world, port, errq):
    """bs_kv_send_layer (rank 0) -> bs_kv_recv_layer (rank 1) over the library's NCCL
    communicator; the destination pool holds the source chunks bit for bit."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2510_13223_b200 as bs
        from paper_2510_13223_b200.transport import NcclWire
        shape = synth.Shape(3, 8, 8, 128)
        g = torch.Generator().manual_seed(5)
        src_np = torch.randint(0, 65536, (3, 40, 2, 8, 16, 128), generator=g,
                               dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)
        s = np.array([5, 0, 39, 17, 22], dtype=np.int32)
        t = np.array([49, 3, 2, 20, 0], dtype=np.int32)
        wire = NcclWire(None)
        if rank == 0:
            src = bs.KVPool(3, 40, shape.hkv, shape.d)
            src.data.copy_(torch.from_numpy(src_np.view(np.int16)).view(torch.bfloat16).cuda())
            stg = torch.empty(len(s) * src.chunk_bytes, dtype=torch.uint8, device="cuda")
            bs.kv_send_layer(src, 2, torch.from_numpy(s).cuda(), 1, wire.comm, stg)
        else:
            dst_np = np.full((3, 50, 2, 8, 16, 128), synth.DST_SENTINEL, dtype=np.uint16)
            dst = bs.KVPool(3, 50, shape.hkv, shape.d)
            dst.data.copy_(torch.from_numpy(dst_np.view(np.int16)).view(torch.bfloat16).cuda())
            stg = torch.empty(len(t) * dst.chunk_bytes, dtype=torch.uint8, device="cuda")
            bs.kv_recv_layer(dst, 2, torch.from_numpy(t).cuda(), 0, wire.comm, stg)
            torch.cuda.synchronize()
            ref = dst_np.copy()
            oracle.migrate_layer(src_np, ref, 2, s, t)
            got = dst.data.cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, ref)
        torch.cuda.synchronize()
        dist.barrier()
        wire.close()
        dist.destroy_process_group()
    except Exception:
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


def test_kv_send_recv_layer_between_gpus():
    _need(2)
    _run(_sendrecv_rank, 2, lambda r, port, errq: (r, 2, port, errq))
