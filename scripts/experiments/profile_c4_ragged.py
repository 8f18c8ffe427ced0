#!/usr/bin/env python
"""A few launches of the C4 per-GPU shard through the packed ragged plan (decode-step flags),
for ncu captures (-k regex:split_decode -s 2 -c 1)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
shape = synth.LLAMA2_70B
lens = np.asarray(synth.mixed_lengths(256, seed=0) // 8, dtype=np.int64)
ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
case = synth.device_shards(shape, lens, ks, seed=1, device=dev, layers=1)
pool = bs.KVPool(1, case.pools[0].shape[1], shape.hkv, shape.d, base=case.pools[0].reshape(-1))
bts = [torch.from_numpy(case.block_tables[0]).to(dev)]
ksd = torch.from_numpy(ks).to(dev)
B = len(lens)
pl = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d, pack_short=True).to(dev)
ws = torch.zeros(max(16, pl.workspace_bytes), dtype=torch.uint8, device=dev)
o = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)
lse = torch.empty(B, shape.hq, device=dev)
for i in range(4):
    bs.split_decode_attention_local_ragged([pool], 0, case.q[0], bts, [0], ksd, synth.default_scale(shape.d),
                                           pl, o, lse, ws, flags=bs.ATTN_PDL if i else 0)
torch.cuda.synchronize()
print("ok", pl.n_work)
