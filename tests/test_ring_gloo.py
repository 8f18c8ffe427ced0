"""Multi-instance protocol (paper_2510_13223_b200/ring.py) on CPU under gloo, world sizes
1, 2 and 3: the same ShardedDecodeStep code the GPU bench runs, with the oracle as the
kernels (test infrastructure) and gloo as the transport.  Checks, on every rank:
  * merged O / lse of the rank's own requests == oracle attention over the whole KV,
    although shard 1 lived on the next rank and its partial came back over the wire;
  * hand-off chunks received from the next rank landed bit-exact in the home pool;
  * H7: each request's decoded-token K/V (sent with q to the rank holding the end of its
    shard 1 and appended there) is part of the KV the attention saw."""
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
from paper_2510_13223_b200.ring import CpuExec, ShardedDecodeStep, split_partial

SHAPE = synth.Shape(2, 4, 2, 64)
LENS = (37, 64, 100)
N_HANDOFF_BLOCKS = 5


def lens_of(rank):
    """Every rank has the same batch size but its own lengths (so its own split points:
    the cold instance must index its predecessor's requests with the predecessor's split)."""
    return tuple(n + 17 * rank for n in LENS)


class NpPool:
    def __init__(self, arr):
        self.data = arr  # uint16 [L][NB][2][Hkv][16][d]


class OracleOps:
    """Kernels for the CPU protocol test: the fp64 oracle (test infrastructure only)."""

    def __init__(self, scale):
        self.scale = scale

    @staticmethod
    def _u16(t):
        return t.contiguous().view(torch.int16).numpy().view(np.uint16)

    def attention(self, pool, layer, q, bt, ks, shard, part):
        o, m, l = oracle.attention_shard(pool.data, layer, self._u16(q), bt, ks, shard, self.scale)
        part[0].copy_(torch.from_numpy(o))
        part[1].copy_(torch.from_numpy(m))
        part[2].copy_(torch.from_numpy(l))

    def merge(self, parts, out, lse):
        o, x = oracle.merge_partials([p[0].double().numpy() for p in parts],
                                     [p[1].double().numpy() for p in parts],
                                     [p[2].double().numpy() for p in parts])
        out.copy_(torch.from_numpy(o).to(torch.bfloat16))
        lse.copy_(torch.from_numpy(x))

    def append(self, pool, layer, k_new, v_new, bt, pos):
        oracle.append_token(pool.data, layer, self._u16(k_new), self._u16(v_new), bt, pos.numpy())

    def migrate_local(self, src, dst, layer, s, d, host_ids=None):
        oracle.migrate_layer(src.data, dst.data, layer, s.numpy(), d.numpy())

    def gather(self, pool, layer, ids, staging):
        chunks = pool.data[layer, ids.numpy()]
        staging[: chunks.nbytes].copy_(torch.from_numpy(chunks.reshape(-1).view(np.uint8)))

    def scatter(self, pool, layer, ids, staging):
        n = len(ids)
        c = pool.data[layer, 0].size
        arr = staging[: n * c * 2].numpy().view(np.uint16).reshape((n,) + pool.data.shape[2:])
        pool.data[layer, ids.numpy()] = arr

    def partial_buffers(self, pool, B, hq, d, max_blocks, device):
        flat = torch.zeros(B * hq * (d + 2), dtype=torch.float32)
        return split_partial(flat, B, hq, d) + (None, flat)


def handoff_bytes(owner_seed):
    """KV the cold pool of rank `owner` hands off to its prev: seeded random bits."""
    g = torch.Generator().manual_seed(1000 + owner_seed)
    shp = (SHAPE.n_layers, N_HANDOFF_BLOCKS, 2, SHAPE.hkv, SHAPE.bs, SHAPE.d)
    return torch.randint(0, 65536, shp, generator=g, dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def rank_setup(rank, world):
    prev, nxt = (rank - 1) % world, (rank + 1) % world
    ks = synth.block_aligned_split(lens_of(rank), 2)
    ks_prev = synth.block_aligned_split(lens_of(prev), 2)
    own = synth.gen_dense(SHAPE, lens_of(rank), seed=rank)
    prv = synth.gen_dense(SHAPE, lens_of(prev), seed=prev)
    home = synth.place_shards(own, ks, seed=rank, spare_blocks=N_HANDOFF_BLOCKS + 2)[0]
    cold = synth.place_shards(prv, ks_prev, seed=prev, spare_blocks=N_HANDOFF_BLOCKS + 2)[1]
    free_home = [i for i in range(home.pool.shape[1]) if not home.used[i]][:N_HANDOFF_BLOCKS]
    free_cold = [i for i in range(cold.pool.shape[1]) if not cold.used[i]][:N_HANDOFF_BLOCKS]
    cold.pool[:, free_cold] = handoff_bytes(rank)       # what I hand off to prev
    return own, ks, home, cold, free_home, free_cold, nxt


def run_rank(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        if world > 1:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        own, ks, home, cold, free_home, free_cold, nxt = rank_setup(rank, world)
        sc = synth.default_scale(SHAPE.d)
        hp, cp = NpPool(home.pool), NpPool(cold.pool)
        # H7: the decoded token's K/V of my requests (random), appended at the end of their
        # shard 1 -- on the next rank, which receives them with q
        gk = torch.Generator().manual_seed(99 + rank)
        kv_new = torch.randn((SHAPE.n_layers, 2, len(LENS), SHAPE.hkv, SHAPE.d),
                             generator=gk).to(torch.bfloat16)
        step = ShardedDecodeStep(
            OracleOps(sc), CpuExec(), rank, world, hp, home.block_tables, cp, cold.block_tables,
            ks, SHAPE.hq, SHAPE.n_layers, SHAPE.d,
            handoff_src_ids=torch.tensor(free_cold, dtype=torch.int64),
            handoff_dst_ids=torch.tensor(free_home, dtype=torch.int64),
            chunk_bytes=oracle.chunk_elems(SHAPE.hkv, 16, SHAPE.d) * 2,
            pg_attn=dist.group.WORLD if world > 1 else None,
            pg_mig=dist.new_group(list(range(world))) if world > 1 else None, append=kv_new,
            wire_attn=GlooWire() if world > 1 else None, wire_mig=GlooWire() if world > 1 else None)
        q = torch.from_numpy(own.q.view(np.int16)).view(torch.bfloat16)
        out = torch.zeros(q.shape, dtype=torch.bfloat16)
        lse = torch.zeros(q.shape[:-1], dtype=torch.float32)
        step.enqueue(q, out, lse)
        # reference: the rank's own requests over their whole KV (both shards), ending with
        # the appended token
        bits = kv_new.view(torch.int16).numpy().view(np.uint16)
        for b, n in enumerate(lens_of(rank)):
            own.k[b][:, n - 1] = bits[:, 0, b]
            own.v[b][:, n - 1] = bits[:, 1, b]
        for layer in range(SHAPE.n_layers):
            shards = synth.place_shards(own, ks, seed=rank)
            ref_o, ref_lse = oracle.attention_full([s.pool for s in shards],
                                                   [s.block_tables for s in shards], layer,
                                                   own.q[layer], ks, sc)
            got = out[layer].float().double().numpy()
            assert np.abs(got - ref_o).max() <= 2e-2, (rank, layer)
            assert np.abs(lse[layer].double().numpy() - ref_lse).max() <= 1e-5, (rank, layer)
        # hand-offs from the next rank landed bit-exact in my home pool
        exp = handoff_bytes(nxt)
        assert np.array_equal(hp.data[:, free_home], exp), rank
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        import traceback
        errq.put(f"rank {rank}: {traceback.format_exc()}")
        raise


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ring_world1_closes_on_itself():
    import queue
    q = queue.Queue()
    run_rank(0, 1, free_port(), q)
    assert q.empty()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_gloo(world):
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
