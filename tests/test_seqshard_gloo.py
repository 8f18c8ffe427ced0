"""Sequence-sharded step (paper_2510_13223_b200/seqshard.py, SURVEY.md §8(e) partitioning
for C3 / C4) on CPU under gloo, world sizes 1..4, collective transport, with the oracle
as the kernels (test infrastructure).  Every request's KV is split W ways (range r on
rank r; random block-aligned cuts incl. empty ranges); request i's home is rank i mod W.
Checks on every rank: merged O / lse of its home requests == oracle attention over the
whole KV (the other W-1 partials came over the wire), and the hand-off chunks pushed by
the previous rank landed bit-exact in its pool."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from gloo_wire import GlooWire
from paper_2510_13223_b200.seqshard import SeqShardedStep

from test_ring_gloo import NpPool, OracleOps  # noqa: E402  (test-infrastructure kernels)

SHAPE = synth.Shape(2, 8, 2, 64)
LENS = (37, 300, 0, 129, 64, 1, 250, 96, 17, 200, 48, 33)   # 12 requests: W in {1,2,3,4}
N_HANDOFF = 3


def handoff_bytes(owner):
    g = torch.Generator().manual_seed(2000 + owner)
    shp = (SHAPE.n_layers, N_HANDOFF, 2, SHAPE.hkv, SHAPE.bs, SHAPE.d)
    return torch.randint(0, 65536, shp, generator=g, dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def setup(rank, world):
    ks = synth.random_split(LENS, world, seed=world)
    ks = (ks // 16) * 16
    ks[:, -1] = np.asarray(LENS)                 # block-aligned cuts, exact ends
    ks[:, 0] = 0
    ks = np.maximum.accumulate(ks, axis=1).astype(np.int32)
    dense = synth.gen_dense(SHAPE, LENS, seed=7)
    shards = synth.place_shards(dense, ks, seed=7, spare_blocks=2 * N_HANDOFF + 1)
    mine = shards[rank]
    free = [i for i in range(mine.pool.shape[1]) if not mine.used[i]]
    src, dst = free[:N_HANDOFF], free[N_HANDOFF:2 * N_HANDOFF]
    mine.pool[:, src] = handoff_bytes(rank)
    return dense, ks, shards, mine, src, dst


def run_rank(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        if world > 1:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        dense, ks, shards, mine, src, dst = setup(rank, world)
        sc = synth.default_scale(SHAPE.d)
        pool = NpPool(mine.pool)
        step = SeqShardedStep(OracleOps(sc), rank, world, pool, torch.from_numpy(mine.block_tables),
                              torch.from_numpy(ks), SHAPE.hq, SHAPE.n_layers, SHAPE.d, SHAPE.hkv,
                              group=dist.group.WORLD if world > 1 else None, transport="collective",
                              handoff_src_ids=torch.tensor(src), handoff_dst_ids=torch.tensor(dst),
                              wire=GlooWire() if world > 1 else None)
        assert step.transport == "collective"
        q_all = torch.from_numpy(dense.q.view(np.int16)).view(torch.bfloat16)
        q = q_all[:, rank::world].contiguous()
        out = torch.zeros(q.shape, dtype=torch.bfloat16)
        lse = torch.zeros(q.shape[:-1], dtype=torch.float32)
        step.enqueue(q, out, lse)
        ref_shards = synth.place_shards(dense, ks, seed=7)
        for layer in range(SHAPE.n_layers):
            ref_o, ref_lse = oracle.attention_full([s.pool for s in ref_shards],
                                                   [s.block_tables for s in ref_shards], layer,
                                                   dense.q[layer], ks, sc)
            got = out[layer].float().double().numpy()
            assert np.abs(got - ref_o[rank::world]).max() <= 2e-2, (rank, layer)
            gl, rl = lse[layer].double().numpy(), ref_lse[rank::world]
            fin = np.isfinite(rl)
            assert np.array_equal(np.isneginf(gl), ~fin)
            assert np.abs(gl[fin] - rl[fin]).max() <= 1e-5, (rank, layer)
        prev = (rank - 1) % world
        assert np.array_equal(pool.data[:, dst], handoff_bytes(prev)), rank
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
    except Exception:
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_seqshard_world1():
    import queue
    q = queue.Queue()
    run_rank(0, 1, free_port(), q)
    assert q.empty()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_seqshard_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=run_rank, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
