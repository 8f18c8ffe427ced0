#!/usr/bin/env python
"""Task launch (bs_split_decode_attention_tasks) over a C4-shaped mixed-length shard: request
dispatch order = identity vs longest first (bs_attn_task.order), graph-timed (20 launches)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    for seed in (0, 3):
        shape = synth.LLAMA2_70B
        lens = np.asarray(synth.mixed_lengths(256, seed=seed) // 8, dtype=np.int64)
        ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
        case = synth.device_shards(shape, lens, ks, seed=1, device=dev, layers=1)
        pool = bs.KVPool(1, case.pools[0].shape[1], shape.hkv, shape.d, base=case.pools[0].reshape(-1))
        bt = torch.from_numpy(case.block_tables[0]).to(dev)
        ksd = torch.from_numpy(ks).to(dev)
        B = len(lens)
        n = bs.attention_problem_workspace_size(B, shape.hq, shape.hkv, shape.d, [bt.shape[1]])
        ws = torch.zeros(max(n, 16), dtype=torch.uint8, device=dev)
        out = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(B, shape.hq, device=dev)
        order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
        prob = {"q": case.q[0], "kv_split": ksd, "max_blocks": [bt.shape[1]], "out": out, "lse": lse,
                "workspace": ws, "done": None, "cross_device": False}
        for name, o in (("identity", None), ("longest_first", order)):
            def launch():
                bs.split_decode_attention_tasks([prob], [(pool, bt, 0, 0, o)], 0, B, shape.hq,
                                                synth.default_scale(shape.d))
            launch()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            with torch.cuda.graph(g, stream=st):
                for _ in range(20):
                    launch()
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
            print(json.dumps({"case": f"C4_gqa8_mixed_B256_seed{seed}", "order": name, "us": round(us, 2),
                              "kv_GBps": round(kv / (us * 1e-6) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
