#!/usr/bin/env python
"""Small launches of the cluster-merge and PDL paths for compute-sanitizer:

    compute-sanitizer --tool racecheck python scripts/sanitize_cluster.py

Every launch is checked to take the path it is meant for (bs_attention_last_launch)."""
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
    seen = set()
    for (d, G, lens) in ((128, 4, (3000, 0, 1, 17, 999, 2048)), (64, 8, (2000, 5, 700, 1, 64, 90)),
                         (128, 1, (1500, 33, 0, 16, 400, 1000))):
        shape = synth.Shape(2, 8 * G, 8, d)
        dense = synth.gen_dense(shape, lens, seed=1)
        ks = synth.random_split(lens, 2, seed=2)
        shards = synth.place_shards(dense, ks, seed=3)
        pools = []
        for s in shards:
            p = bs.KVPool(2, s.pool.shape[1], 8, d)
            p.data.copy_(dev_bf16(s.pool))
            pools.append(p)
        bts = [torch.from_numpy(s.block_tables).cuda() for s in shards]
        ksd = torch.from_numpy(ks).cuda()
        B, hq = len(lens), shape.hq
        ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
            pools, [t.shape[1] for t in bts], B, hq)), dtype=torch.uint8, device="cuda")
        out = torch.empty(2, B, hq, d, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(2, B, hq, device="cuda")
        for layer in range(2):   # layer 1: a programmatic dependent of layer 0
            bs.split_decode_attention_local(pools, layer, dev_bf16(dense.q[layer]), bts, [0, 1], ksd,
                                            synth.default_scale(d), out[layer], lse[layer], ws,
                                            flags=bs.ATTN_PDL if layer else 0)
            info = bs.attention_last_launch()
            assert info["cluster"] == (1 if 2 <= info["ranges"] <= 8 else 0), info
            seen.add(("G", G, "d", d, "ranges", info["ranges"], "cluster", info["cluster"], "pdl", info["pdl"]))
        torch.cuda.synchronize()
    # one CTA per SM (C3 B=1 shape, shortened): PDL with the late trigger, workspace merge
    shape = synth.Shape(2, 32, 8, 128)
    lens = np.full(1, 4096)
    ks = np.stack([np.zeros(1), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=9, device="cuda")
    pools = [bs.KVPool(2, p.shape[1], 8, 128, base=p.reshape(-1)) for p in case.pools]
    bts = [torch.from_numpy(b).cuda() for b in case.block_tables]
    ksd = torch.from_numpy(ks).cuda()
    ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(pools, [bts[0].shape[1]], 1, 32)),
                     dtype=torch.uint8, device="cuda")
    out = torch.empty(2, 1, 32, 128, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(2, 1, 32, device="cuda")
    for layer in range(2):
        bs.split_decode_attention_local(pools, layer, case.q[layer], bts, [0], ksd, synth.default_scale(128),
                                        out[layer], lse[layer], ws, flags=bs.ATTN_PDL if layer else 0)
        info = bs.attention_last_launch()
        seen.add(("one_per_sm", info["ranges"], info["pdl"], info["cluster"]))
    torch.cuda.synchronize()
    print("sanitize_cluster: paths", sorted(seen))


if __name__ == "__main__":
    main()
