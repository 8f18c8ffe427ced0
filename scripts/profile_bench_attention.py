#!/usr/bin/env python
"""Launch the bench's per-layer attention exactly as bench.py does (C2, N=1: fused local
shards over the home and cold pools) for a few layers, for ncu captures.

    ncu --set full -k regex:split_decode -s 2 -c 1 -o out python scripts/profile_bench_attention.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2510_13223_b200 as bs  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
case, pools, step, ks = bench.build_workload(bs, dev, 0, 1, layers=4)
L = 4
out = torch.empty((L,) + tuple(case.q.shape[1:]), dtype=torch.bfloat16, device=dev)
lse = torch.empty(out.shape[:-1], dtype=torch.float32, device=dev)
for _ in range(2):
    step.enqueue(case.q, out, lse)
torch.cuda.synchronize()
print("ok", step.launches_per_step)
