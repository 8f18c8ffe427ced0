#!/usr/bin/env python
"""SM clock and board power of the C2 step's parts (power-capped boxes): the full step, the
step without the hand-off, and the hand-off copies alone -- each replayed from a CUDA graph
for ~2 s with the bench's NVML sampler."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_13223_b200 as bs  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    case, pools, step, ks = bench.build_workload(bs, dev)
    L = bench.SHAPE.n_layers
    out = torch.empty((L, bench.BATCH, bench.SHAPE.hq, bench.SHAPE.d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((L, bench.BATCH, bench.SHAPE.hq), dtype=torch.float32, device=dev)
    n_hand = step.n_handoff

    def mig_only():
        for layer in range(L):
            step.ops.migrate_local(step.cold, step.home, layer, step.src_ids, step.dst_ids, step.ce_ids)

    variants = {"full_step": lambda: step.enqueue(case.q, out, lse), "no_handoff": None, "handoff_only": mig_only}
    res = {}
    for name in ("full_step", "no_handoff", "handoff_only", "full_step"):
        step.n_handoff = 0 if name == "no_handoff" else n_hand
        fn = variants[name] or (lambda: step.enqueue(case.q, out, lse))
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                fn()
        g.replay()
        torch.cuda.synchronize()
        reps = 0
        with bench.ClockSampler(0) as clk:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            while reps < 20:
                g.replay()
                reps += 1
            e1.record()
            torch.cuda.synchronize()
        c = clk.summary()
        res.setdefault(name, []).append({"ms_per_iter": round(e0.elapsed_time(e1) / (reps * 10), 4),
                                         "sm_mhz": c["sm_mhz"], "power_w_median": c.get("power_w_median"),
                                         "power_w_max": c.get("power_w_max"), "reasons": c["reasons"]})
        del g
    step.n_handoff = n_hand
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
