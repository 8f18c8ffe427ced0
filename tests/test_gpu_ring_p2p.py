"""The N>1 ring on real GPU kernels with the P2P transport (CUDA IPC pushes + flags),
run as 2 and 3 processes sharing GPU 0 (the only GPU gpurun offers; IPC between
processes works on one device, NCCL does not).  Every rank checks its merged O / lse
against the oracle over its requests' whole KV (shard 1 lived on the next rank) and the
hand-off chunks pushed into its home pool by the next rank, over two steps (epochs) so
the back-pressure acks are exercised.  The graph variant then captures the step in a CUDA
graph on every rank (flags computed on the device from the step counter) and checks that
two replays reproduce the eager outputs bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu

SHAPE = synth.Shape(2, 8, 2, 128)
LENS = (37, 64, 300)
N_HANDOFF_BLOCKS = 5


def lens_of(rank):
    """Every rank has the same batch size but its own lengths (so its own split points:
    the cold instance must index its predecessor's requests with the predecessor's split)."""
    return tuple(n + 17 * rank for n in LENS)


def handoff_bytes(owner_seed):
    g = torch.Generator().manual_seed(1000 + owner_seed)
    shp = (SHAPE.n_layers, N_HANDOFF_BLOCKS, 2, SHAPE.hkv, SHAPE.bs, SHAPE.d)
    return torch.randint(0, 65536, shp, generator=g, dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def run_rank(rank, world, port, errq, fused, graph=False, cross=False, transport="p2p"):
    """cross: rank r on cuda:r (distinct GPUs: NVLink / peer mappings); else every rank on
    cuda:0.  transport "nccl": the library's own NCCL communicator (distinct GPUs only)."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank if cross else 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2510_13223_b200 as bs
        from paper_2510_13223_b200.ring import CudaExec, CudaOps, ShardedDecodeStep
        prev, nxt = (rank - 1) % world, (rank + 1) % world
        ks = synth.block_aligned_split(lens_of(rank), 2)
        ks_prev = synth.block_aligned_split(lens_of(prev), 2)
        own = synth.gen_dense(SHAPE, lens_of(rank), seed=rank)
        prv = synth.gen_dense(SHAPE, lens_of(prev), seed=prev)
        home = synth.place_shards(own, ks, seed=rank, spare_blocks=N_HANDOFF_BLOCKS + 2)[0]
        cold = synth.place_shards(prv, ks_prev, seed=prev, spare_blocks=N_HANDOFF_BLOCKS + 2)[1]
        free_home = [i for i in range(home.pool.shape[1]) if not home.used[i]][:N_HANDOFF_BLOCKS]
        free_cold = [i for i in range(cold.pool.shape[1]) if not cold.used[i]][:N_HANDOFF_BLOCKS]
        cold.pool[:, free_cold] = handoff_bytes(rank)
        hp = bs.KVPool(SHAPE.n_layers, home.pool.shape[1], SHAPE.hkv, SHAPE.d)
        hp.data.copy_(_dev(home.pool))
        cp = bs.KVPool(SHAPE.n_layers, cold.pool.shape[1], SHAPE.hkv, SHAPE.d)
        cp.data.copy_(_dev(cold.pool))
        i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32).cuda()
        dev = torch.device("cuda", rank if cross else 0)
        sc = synth.default_scale(SHAPE.d)
        # H7: each request's decoded token K/V, pushed with q to the next rank, which
        # appends it at the end of shard 1 in its cold pool before attention
        gk = torch.Generator(device="cuda")
        gk.manual_seed(99 + rank)
        kv_new = torch.randn((SHAPE.n_layers, 2, len(LENS), SHAPE.hkv, SHAPE.d), generator=gk,
                             device="cuda", dtype=torch.bfloat16)
        step = ShardedDecodeStep(CudaOps(sc), CudaExec(dev), rank, world, hp, i32(home.block_tables),
                                 cp, i32(cold.block_tables), i32(ks), SHAPE.hq, SHAPE.n_layers, SHAPE.d,
                                 handoff_src_ids=i32(free_cold), handoff_dst_ids=i32(free_home),
                                 chunk_bytes=hp.chunk_bytes, pg_attn=dist.group.WORLD,
                                 pg_mig=dist.new_group(list(range(world))),
                                 device=dev, transport=transport, fused_exchange=fused, append=kv_new)
        assert step.transport == transport, getattr(step, "fallback_reason", None)
        assert step.fused_exchange == (fused and transport == "p2p")
        q = _dev(own.q)
        for _ in range(2):   # two epochs
            out = torch.full(q.shape, float("nan"), dtype=torch.bfloat16, device=dev)
            lse = torch.full(q.shape[:-1], float("nan"), device=dev)
            step.enqueue(q, out, lse)
            torch.cuda.synchronize()
            if step.links is not None:
                step.links.check()
            dist.barrier()
            bits = kv_new.cpu().view(torch.int16).numpy().view(np.uint16)  # the reference KV
            for b, n in enumerate(lens_of(rank)):                          # ends with the
                own.k[b][:, n - 1] = bits[:, 0, b]                         # appended token
                own.v[b][:, n - 1] = bits[:, 1, b]
            shards = synth.place_shards(own, ks, seed=rank)
            for layer in range(SHAPE.n_layers):
                ref_o, ref_lse = oracle.attention_full([s.pool for s in shards],
                                                       [s.block_tables for s in shards], layer,
                                                       own.q[layer], ks, sc)
                got = out[layer].float().cpu().double().numpy()
                assert np.abs(got - ref_o).max() <= 2e-2, (rank, layer)
                assert np.abs(lse[layer].cpu().double().numpy() - ref_lse).max() <= 1e-4, (rank, layer)
        if graph:  # the captured step replays the eager one bit for bit
            ref_out, ref_lse = out.clone(), lse.clone()
            out.fill_(float("nan"))
            lse.fill_(float("nan"))
            g = step.capture(q, out, lse)
            for _ in range(2):
                out.fill_(float("nan"))
                g.replay()
                torch.cuda.synchronize()
                step.links.check()
                assert torch.equal(out.view(torch.int16), ref_out.view(torch.int16)), rank
                assert torch.equal(lse, ref_lse), rank
            dist.barrier()
        got_home = hp.data.cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got_home[:, free_home], handoff_bytes(nxt)), rank
        dist.barrier()
        step.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
@pytest.mark.parametrize("fused", [True, False], ids=["fused-exchange", "push-partials"])
@pytest.mark.parametrize("world", [2, 3])
def test_ring_p2p_on_one_gpu(world, fused, graph):
    if graph and world == 3:
        pytest.skip("graph replay: 2 ranks suffice")
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=run_rank, args=(r, world, port, errq, fused, graph))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not alive, "ranks hung"
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
