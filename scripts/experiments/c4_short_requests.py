#!/usr/bin/env python
"""How much do C4's short requests cost?  The C4 per-GPU shard through the ragged plan with
decode-step flags (graph, 20 launches): all 256 requests vs only those with >= 16 blocks in
this shard vs only the short ones; reports us and KV GB/s of each."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402


def time_ragged(shape, lens, dev, pack=False):
    lens = np.asarray(lens, dtype=np.int64)
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=1, device=dev, layers=1)
    pool = bs.KVPool(1, case.pools[0].shape[1], shape.hkv, shape.d, base=case.pools[0].reshape(-1))
    bts = [torch.from_numpy(case.block_tables[0]).to(dev)]
    ksd = torch.from_numpy(ks).to(dev)
    B = len(lens)
    sc = synth.default_scale(shape.d)
    o = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, shape.hq, device=dev)
    pl = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d, pack_short=pack).to(dev)
    ws = torch.zeros(max(16, pl.workspace_bytes), dtype=torch.uint8, device=dev)

    def launch(flags):
        bs.split_decode_attention_local_ragged([pool], 0, case.q[0], bts, [0], ksd, sc, pl, o, lse, ws,
                                               flags=flags)
    launch(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            launch(bs.ATTN_PDL if i else 0)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 20)
    us = sorted(ts)[5] * 1e3
    kv = int(lens.sum()) * 2 * shape.hkv * shape.d * 2
    return round(us, 2), round(kv / (us * 1e-6) / 1e9, 1), B, int(lens.sum())


def main():
    dev = torch.device("cuda")
    shape = synth.LLAMA2_70B
    for seed in (0, 3):
        lens = synth.mixed_lengths(256, seed=seed) // 8
        for name, sel, pack in (("all", lens, False), ("all_packed", lens, True),
                                ("long_ge16blocks", lens[lens >= 256], False),
                                ("short_lt16blocks", lens[lens < 256], False),
                                ("short_lt16blocks_packed", lens[lens < 256], True)):
            us, gbps, B, tok = time_ragged(shape, sel, dev, pack)
            print(json.dumps({"seed": seed, "subset": name, "requests": B, "tokens": tok, "us": us, "kv_GBps": gbps}),
                  flush=True)


if __name__ == "__main__":
    main()
