#!/usr/bin/env python
"""Experiment: does per-kernel event instrumentation perturb the C2 step?  Times K steps
of the N=1 bench step five ways: graph untimed / graph with attention-only timers / graph
with every timer / eager untimed / eager with every timer (alternating, 3 rounds)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_13223_b200 as bs  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
case, pools, step, ks = bench.build_workload(bs, dev)
L, K = 32, 20
q = case.q
out = torch.empty((L, 64, 32, 128), dtype=torch.bfloat16, device=dev)
lse = torch.empty((L, 64, 32), dtype=torch.float32, device=dev)
for _ in range(3):
    step.enqueue(q, out, lse)
torch.cuda.synchronize()


class Attn2:  # only the attention pair of a layer's timers is real
    def __init__(self):
        self.t = [bench.DrvTimer(), bench.DrvTimer()]
        self.n = _Null()

    def __getitem__(self, i):
        return self.t[i] if i < 2 else self.n

    def __len__(self):
        return 4


class _Null:
    def record(self, *a):
        pass


def graph_of(timers):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k in range(K):
            step.enqueue(q, out, lse, **({} if timers is None else {"timers": timers[k]}))
    torch.cuda.synchronize()
    return g


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


full = [[tuple(bench.DrvTimer() for _ in range(5)) for _ in range(L)] for _ in range(K)]
attn = [[Attn2() for _ in range(L)] for _ in range(K)]
g0, g1, g2 = graph_of(None), graph_of(attn), graph_of(full)
res = {k: [] for k in ("graph_untimed", "graph_attn_timers", "graph_all_timers", "eager_untimed",
                       "eager_all_timers")}
for _ in range(3):
    res["graph_untimed"].append(timeit(g0.replay))
    res["graph_attn_timers"].append(timeit(g1.replay))
    res["graph_all_timers"].append(timeit(g2.replay))
    res["eager_untimed"].append(timeit(lambda: [step.enqueue(q, out, lse) for _ in range(K)]))
    res["eager_all_timers"].append(timeit(lambda: [step.enqueue(q, out, lse, timers=full[k])
                                                   for k in range(K)]))
a = [t[0].elapsed_time(t[1]) for tk in attn for t in tk]
res["attn_ms_per_layer_attn_timers"] = sum(a) / len(a)
b = [t[0].elapsed_time(t[1]) for tk in full for t in tk]
res["attn_ms_per_layer_all_timers_eager"] = sum(b) / len(b)
print(json.dumps(res))
