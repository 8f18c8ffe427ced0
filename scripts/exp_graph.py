#!/usr/bin/env python
"""Experiment: eager submission vs CUDA-graph replay of the N=1 bench step (no timers)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2510_13223_b200 as bs  # noqa: E402


def timed(fn, K):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def main():
    dev = torch.device("cuda", 0)
    case, pools, step, ks = bench.build_workload(bs, dev)
    L = bench.SHAPE.n_layers
    out = torch.empty((L, bench.BATCH, bench.SHAPE.hq, bench.SHAPE.d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((L, bench.BATCH, bench.SHAPE.hq), dtype=torch.float32, device=dev)
    g = step.capture(case.q, out, lse)
    res = {}
    for rep in range(3):
        res[f"eager_{rep}"] = timed(lambda: step.enqueue(case.q, out, lse), 20)
        res[f"graph_{rep}"] = timed(g.replay, 20)
    print(json.dumps({k: round(v, 4) for k, v in res.items()}))


if __name__ == "__main__":
    main()
