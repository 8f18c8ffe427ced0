#!/usr/bin/env python
"""Small launches of every kernel for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def main():
    for (d, G) in ((64, 2), (128, 8), (128, 1)):
        shape = synth.Shape(1, 2 * G, 2, d)
        lens = (0, 1, 17, 300)
        dense = synth.gen_dense(shape, lens, seed=1)
        ks = synth.random_split(lens, 2, seed=2)
        shards = synth.place_shards(dense, ks, seed=3)
        pools = []
        for s in shards:
            p = bs.KVPool(1, s.pool.shape[1], 2, d)
            p.data.copy_(dev_bf16(s.pool))
            pools.append(p)
        bts = [torch.from_numpy(s.block_tables).cuda() for s in shards]
        ksd = torch.from_numpy(ks).cuda()
        q = dev_bf16(dense.q[0])
        B, hq = len(lens), shape.hq
        parts = []
        for j, (p, bt) in enumerate(zip(pools, bts)):
            o = torch.empty(B, hq, d, device="cuda")
            m = torch.empty(B, hq, device="cuda")
            l = torch.empty(B, hq, device="cuda")
            ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(p, B, hq, bt.shape[1])),
                             dtype=torch.uint8, device="cuda")
            bs.split_decode_attention(p, 0, q, bt, ksd, j, synth.default_scale(d), o, m, l, ws)
            parts.append((o, m, l))
        out = torch.empty(B, hq, d, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(B, hq, device="cuda")
        bs.merge_partials([x[0] for x in parts], [x[1] for x in parts], [x[2] for x in parts], out, lse)
        ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
            pools, [t.shape[1] for t in bts], B, hq)), dtype=torch.uint8, device="cuda")
        bs.split_decode_attention_local(pools, 0, q, bts, [0, 1], ksd, synth.default_scale(d), out, lse, ws)
        # ragged plan over the same local shards
        plan = bs.attention_ragged_plan(ks, [0, 1], hq, 2, d, max_blocks_per_range=16).to("cuda")
        wsr = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device="cuda")
        bs.split_decode_attention_local_ragged(pools, 0, q, bts, [0, 1], ksd, synth.default_scale(d),
                                               plan, out, lse, wsr)
        # tasks: the same problem cut over two launches (stand-ins for two GPUs), sys scope
        mb = [t.shape[1] for t in bts]
        wst = torch.zeros(max(256, bs.attention_problem_workspace_size(B, hq, 2, d, mb)),
                          dtype=torch.uint8, device="cuda")
        done = torch.zeros(1, dtype=torch.int32, device="cuda")
        prob = {"q": q, "kv_split": ksd, "max_blocks": mb, "out": out, "lse": lse, "workspace": wst,
                "done": done, "cross_device": True}
        for j in range(2):
            bs.split_decode_attention_tasks([prob], [(pools[j], bts[j], j, 0)], 0, B, hq,
                                            synth.default_scale(d))
        # one long request: intra-GPU split-K over up to 64 ranges (the merge's unrolled
        # 16-deep loads plus remainder, and its cross-thread-group reduction for G*D < 512)
        lg = synth.gen_dense(shape, (8192,), seed=4)
        kl = np.array([[0, 8192]], dtype=np.int32)
        sl = synth.place_shards(lg, kl, seed=5)[0]
        pl_ = bs.KVPool(1, sl.pool.shape[1], 2, d)
        pl_.data.copy_(dev_bf16(sl.pool))
        btl = torch.from_numpy(sl.block_tables).cuda()
        o = torch.empty(1, hq, d, device="cuda")
        m = torch.empty(1, hq, device="cuda")
        l = torch.empty(1, hq, device="cuda")
        wsl = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pl_, 1, hq, btl.shape[1])),
                          dtype=torch.uint8, device="cuda")
        bs.split_decode_attention(pl_, 0, dev_bf16(lg.q[0]), btl, torch.from_numpy(kl).cuda(), 0,
                                  synth.default_scale(d), o, m, l, wsl)
        # migration kernels
        dst = bs.KVPool(1, 64, 2, d)
        ids = torch.tensor([x for x in shards[1].block_tables.ravel() if x >= 0], dtype=torch.int32).cuda()
        tgt = torch.arange(ids.numel(), dtype=torch.int32).cuda()
        for method in (1, 2):
            bs.kv_migrate_layer(pools[1], dst, 0, ids, tgt, method=method)
        cold = bs.KVPool(1, 64, 1, d)
        bs.kv_migrate_heads_layer(dst, cold, 0, tgt, tgt, 1, 0, 1)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
