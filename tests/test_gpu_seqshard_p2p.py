"""Sequence-sharded step with the fused P2P exchange (paper_2510_13223_b200/seqshard.py)
on the real kernels, W = 2, 3, 4 processes sharing GPU 0 (IPC works between processes on
one device).  Every request's KV is split W ways; rank r holds range r of every request
and is home of requests r, r+W, ...; one launch per layer per rank runs shard r of every
home's problem and the last-arriving CTA merges into the home's buffers.
  * toy (two epochs, hand-off chunks pushed to the next rank's pool): merged O / lse of
    each home's requests == oracle over the whole KV; hand-off bytes exact;
  * C3-shaped (Llama-3-8B GQA 32/8, d 128, 32k context, 4-way, B = 8, one layer):
    two sampled requests per home against the oracle."""
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

TOY = synth.Shape(2, 8, 2, 128)
TOY_LENS = (37, 300, 0, 129, 64, 1, 250, 96, 17, 200, 48, 33)
N_HANDOFF = 3


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def handoff_bytes(owner):
    g = torch.Generator().manual_seed(3000 + owner)
    shp = (TOY.n_layers, N_HANDOFF, 2, TOY.hkv, TOY.bs, TOY.d)
    return torch.randint(0, 65536, shp, generator=g, dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def toy_split(world):
    ks = synth.random_split(TOY_LENS, world, seed=world)
    ks = (ks // 16) * 16
    ks[:, 0], ks[:, -1] = 0, np.asarray(TOY_LENS)
    return np.maximum.accumulate(ks, axis=1).astype(np.int32)


def run_toy(rank, world, cross=False, transport="p2p"):
    import paper_2510_13223_b200 as bs
    from paper_2510_13223_b200.ring import CudaOps
    from paper_2510_13223_b200.seqshard import SeqShardedStep
    ks = toy_split(world)
    dense = synth.gen_dense(TOY, TOY_LENS, seed=11)
    shards = synth.place_shards(dense, ks, seed=11, spare_blocks=2 * N_HANDOFF + 1)
    mine = shards[rank]
    free = [i for i in range(mine.pool.shape[1]) if not mine.used[i]]
    src, dst = free[:N_HANDOFF], free[N_HANDOFF:2 * N_HANDOFF]
    mine.pool[:, src] = handoff_bytes(rank)
    pool = bs.KVPool(TOY.n_layers, mine.pool.shape[1], TOY.hkv, TOY.d)
    pool.data.copy_(_dev(mine.pool))
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32).cuda()
    dev = torch.device("cuda", rank if cross else 0)
    sc = synth.default_scale(TOY.d)
    step = SeqShardedStep(CudaOps(sc), rank, world, pool, i32(mine.block_tables), i32(ks), TOY.hq,
                          TOY.n_layers, TOY.d, TOY.hkv, device=dev, group=dist.group.WORLD,
                          transport=transport, handoff_src_ids=i32(src), handoff_dst_ids=i32(dst))
    assert step.transport == transport, step.fallback_reason
    p2p = transport == "p2p"
    q = _dev(dense.q)[:, rank::world].contiguous()
    ref_shards = synth.place_shards(dense, ks, seed=11)
    for epoch in range(2):
        out, lse = step.outputs() if (epoch == 0 and p2p) else (
            torch.full(q.shape, float("nan"), dtype=torch.bfloat16, device=dev),
            torch.full(q.shape[:-1], float("nan"), device=dev))
        step.enqueue(q, out, lse)
        torch.cuda.synchronize()
        step.check()
        dist.barrier()
        for layer in range(TOY.n_layers):
            ref_o, ref_lse = oracle.attention_full([s.pool for s in ref_shards],
                                                   [s.block_tables for s in ref_shards], layer,
                                                   dense.q[layer], ks, sc)
            got = out[layer].float().cpu().double().numpy()
            assert np.abs(got - ref_o[rank::world]).max() <= 2e-2, (rank, layer, epoch)
            gl, rl = lse[layer].cpu().double().numpy(), ref_lse[rank::world]
            fin = np.isfinite(rl)
            assert np.array_equal(np.isneginf(gl), ~fin), (rank, layer)
            assert np.abs(gl[fin] - rl[fin]).max() <= 1e-4, (rank, layer)
        dist.barrier()
    got_pool = pool.data.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got_pool[:, dst], handoff_bytes((rank - 1) % world)), rank
    if not p2p:
        dist.barrier()
        step.close()
        return
    # the step captured in a CUDA graph (device-computed flags) replays the eager outputs
    ref_out, ref_lse = out.clone(), lse.clone()
    g = step.capture(q, out, lse)
    for _ in range(2):
        out.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        step.check()
        assert torch.equal(out.view(torch.int16), ref_out.view(torch.int16)), rank
        assert torch.equal(lse.view(torch.int32), ref_lse.view(torch.int32)), rank
    dist.barrier()
    step.close()


def run_c3(rank, world, cross=False, transport="p2p"):
    import paper_2510_13223_b200 as bs
    from paper_2510_13223_b200.ring import CudaOps
    from paper_2510_13223_b200.seqshard import SeqShardedStep
    shape = synth.Shape(1, 32, 8, 128)
    lens = [32768] * 8
    ks = synth.block_aligned_split(lens, world)
    case = synth.device_shards(shape, np.asarray(lens), ks, seed=41, device="cuda", layers=1)
    pt = case.pools[rank]
    pool = bs.KVPool(1, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    dev = torch.device("cuda", rank if cross else 0)
    sc = synth.default_scale(shape.d)
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32).cuda()
    step = SeqShardedStep(CudaOps(sc), rank, world, pool, i32(case.block_tables[rank]), i32(ks),
                          shape.hq, 1, shape.d, shape.hkv, device=dev, group=dist.group.WORLD,
                          transport="p2p")
    q = case.q[:, rank::world].contiguous()
    out, lse = step.outputs()
    step.enqueue(q, out, lse)
    torch.cuda.synchronize()
    step.check()
    dist.barrier()
    mine = list(range(rank, len(lens), world))
    sample = [mine[0], mine[-1]]
    sp, sbt, sks, sq = synth.extract_requests(case, sample, 0)
    ref_o, ref_lse = oracle.attention_full(sp, sbt, 0, sq, sks, sc)
    rows = [mine.index(i) for i in sample]
    got = out[0, rows].float().cpu().double().numpy()
    err = np.abs(got - ref_o)
    assert err.max() <= 2e-2
    assert (err.max(-1) / np.abs(ref_o).max(-1)).max() <= 1e-2
    assert np.abs(lse[0, rows].cpu().double().numpy() - ref_lse).max() <= 1e-4
    dist.barrier()
    step.close()


def run_rank(fn_name, rank, world, port, errq, cross=False, transport="p2p"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank if cross else 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        {"toy": run_toy, "c3": run_c3}[fn_name](rank, world, cross, transport)
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


def _spawn(fn_name, world, cross=False, transport="p2p"):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=run_rank, args=(fn_name, r, world, port, errq, cross, transport))
             for r in range(world)]
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


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_seqshard_p2p_toy(world):
    _spawn("toy", world)


def test_seqshard_p2p_c3_shape_4way():
    _spawn("c3", 4)
