#!/usr/bin/env python
"""Functional measurement of the W-way sequence-sharded step with the fused cross-GPU
exchange (paper_2510_13223_b200/seqshard.py) at the C3 / C4 shapes, W processes sharing
ONE GPU (the only GPU a round gets): every rank runs its real per-layer launch (range r
of every home's requests, partials into the homes' workspaces over CUDA IPC, last
arriver merges).  Without MPS the W contexts are time-sliced, so the timings are not
performance numbers (neither HBM nor NVLink) -- this checks the protocol end to end at
the full C3 / C4 shapes.

    python scripts/bench_seqshard.py --config c3|c4 [--layers 4 --steps 5 --json out]

c3: Llama-3-8B GQA (32/8, d 128), B = 8 x 32768 tokens, 4-way split (8192 per rank).
c4: Llama-2-70B GQA (64/8, d 128), B = 256 mixed lengths (seed 0), 8-way split, plus a
    per-layer hand-off of 8192 tokens' chunks into the next rank's pool.
Reported: per-rank step time (max over ranks), aggregate algorithmic attention bytes per
step / that time, and tokens/s (decode tokens of all homes / step time)."""
import argparse
import json
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def config(name):
    if name == "c3":
        return synth.Shape(1, 32, 8, 128), np.full(8, 32768), 4, 0
    return synth.Shape(1, 64, 8, 128), synth.mixed_lengths(256, seed=0), 8, 8192 // 16


def run(rank, world, port, args, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_13223_b200 as bs
    from paper_2510_13223_b200.ring import CudaOps
    from paper_2510_13223_b200.seqshard import SeqShardedStep
    shape0, lens, W, n_handoff = config(args.config)
    shape = synth.Shape(args.layers, shape0.hq, shape0.hkv, shape0.d)
    ks = synth.block_aligned_split(lens, W)
    dev = torch.device("cuda", 0)
    my_lens = (ks[:, rank + 1] - ks[:, rank]).astype(np.int64)
    pool_t, bt = synth.device_pool(shape, my_lens, synth.shard_seed(7, rank), dev,
                                   spare_blocks=2 * n_handoff + 1, layers=args.layers)
    pool = bs.KVPool(args.layers, pool_t.shape[1], shape.hkv, shape.d, base=pool_t.reshape(-1))
    used = set(int(x) for x in bt.ravel() if x >= 0)
    free = [i for i in range(pool_t.shape[1]) if i not in used]
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32, device=dev)
    src = i32(free[:n_handoff]) if n_handoff else None
    dst = i32(free[n_handoff:2 * n_handoff]) if n_handoff else None
    step = SeqShardedStep(CudaOps(synth.default_scale(shape.d)), rank, W, pool, i32(bt), i32(ks),
                          shape.hq, args.layers, shape.d, shape.hkv, device=dev,
                          group=dist.group.WORLD, transport="p2p", handoff_src_ids=src,
                          handoff_dst_ids=dst)
    assert step.transport == "p2p", step.fallback_reason
    q = synth.device_q(shape, len(lens), 5, dev, args.layers)[:, rank::W].contiguous()
    out, lse = step.outputs()
    for _ in range(3):
        step.enqueue(q, out, lse)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        step.enqueue(q, out, lse)
    b.record()
    torch.cuda.synchronize()
    step.check()
    ms = a.elapsed_time(b) / args.steps
    t = torch.tensor([ms])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        kv = int(lens.sum()) * 2 * shape.hkv * shape.d * 2 * args.layers
        q_out.put({"config": args.config, "ranks_on_one_gpu": W, "layers": args.layers,
                   "steps": args.steps, "step_ms_max_over_ranks": round(float(t.item()), 4),
                   "kv_bytes_per_step_all_ranks": kv,
                   "aggregate_kv_GBps": round(kv / (float(t.item()) * 1e-3) / 1e9, 1),
                   "tokens_per_s": round(len(lens) / (float(t.item()) * 1e-3), 1),
                   "handoff_chunks_per_layer_per_rank": n_handoff,
                   "note": "W processes time-share one B200 (no MPS: contexts are time-sliced, "
                           "and a rank's flag-wait kernel holds its slice while the peer it "
                           "waits for cannot run), so the rates say nothing about the kernels "
                           "or NVLink; this is a functional check of the fused exchange at full "
                           "shape"})
    dist.barrier()
    step.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c4"], default="c3")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--json")
    args = ap.parse_args()
    W = config(args.config)[2]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    procs = [ctx.Process(target=run, args=(r, W, port, args, q_out)) for r in range(W)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    res = q_out.get(timeout=5)
    print(json.dumps(res))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
