#!/usr/bin/env python
"""Where the e2e step's time goes (experiment): the C2 N=1 step as one CUDA graph per decode
step, the host waiting for the result each time, with / without the per-layer H2D input
copies and D2H output copies -- plus back-to-back replays without the per-step sync.

    python scripts/exp_e2e.py [--steps 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2510_13223_b200 as bs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    case, pools, step, ks = bench.build_workload(bs, dev)
    L = bench.SHAPE.n_layers
    out = torch.empty((L, bench.BATCH, bench.SHAPE.hq, bench.SHAPE.d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((L, bench.BATCH, bench.SHAPE.hq), dtype=torch.float32, device=dev)
    kv0 = step.append
    in_host, in_dev, rowb, q_dev, kv_dev = bench._e2e_buffers(case.q, kv0, L, dev)
    if kv0 is not None:
        step.append = kv_dev
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    lse_host = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    q_ev = [torch.cuda.Event() for _ in range(L)]
    ob, lb = out[0].numel() * out.element_size(), lse[0].numel() * lse.element_size()

    groups = [(0, 1), (1, 4), (4, L)]   # H2D copies of layer ranges, one event each

    def one(with_h2d, with_d2h, grouped=False):
        cur = torch.cuda.current_stream()
        ready = None
        if with_h2d:
            h2d.wait_stream(cur)
            if grouped:
                ready = [None] * L
                for lo, hi in groups:
                    bs.copy_ptr(in_dev.data_ptr() + lo * rowb, in_host.data_ptr() + lo * rowb,
                                (hi - lo) * rowb, stream=h2d)
                    q_ev[lo].record(h2d)
                    ready[lo] = q_ev[lo]
            else:
                for layer in range(L):
                    bs.copy_ptr(in_dev.data_ptr() + layer * rowb, in_host.data_ptr() + layer * rowb,
                                rowb, stream=h2d)
                    q_ev[layer].record(h2d)
                ready = q_ev
        step.enqueue(q_dev, out, lse, inputs_ready=ready)
        if with_d2h:
            for layer in range(L):
                d2h.wait_event(step.out_ready[layer])
                bs.copy_ptr(out_host.data_ptr() + layer * ob, out.data_ptr() + layer * ob, ob, stream=d2h)
                bs.copy_ptr(lse_host.data_ptr() + layer * lb, lse.data_ptr() + layer * lb, lb, stream=d2h)
            cur.wait_stream(d2h)

    res = {}
    for name, h, d, gr in (("step_only", False, False, False), ("h2d_only", True, False, False),
                           ("h2d_grouped", True, False, True), ("d2h_only", False, True, False),
                           ("e2e", True, True, False), ("e2e_grouped", True, True, True)):
        one(h, d, gr)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            one(h, d, gr)
        torch.cuda.synchronize()
        for sync in (True, False):
            for _ in range(3):
                g.replay()
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                g.replay()
                if sync:
                    torch.cuda.current_stream().synchronize()
            e1.record()
            torch.cuda.synchronize()
            res[f"{name}{'_sync' if sync else '_nosync'}_ms"] = round(e0.elapsed_time(e1) / args.steps, 4)
        del g
    # where the e2e step's time goes: event-record nodes in the e2e graph (bench.DrvTimer)
    for name, h, d in (("e2e", True, True), ("step_only", False, False)):
        T = {k: bench.DrvTimer() for k in ("start", "h2d0", "h2d_all", "end")}
        timers = [tuple(bench.DrvTimer() for _ in range(5)) for _ in range(L)]

        def one_t():
            cur = torch.cuda.current_stream()
            T["start"].record(cur)
            ready = None
            if h:
                h2d.wait_stream(cur)
                for layer in range(L):
                    bs.copy_ptr(in_dev.data_ptr() + layer * rowb, in_host.data_ptr() + layer * rowb,
                                rowb, stream=h2d)
                    q_ev[layer].record(h2d)
                    if layer == 0:
                        T["h2d0"].record(h2d)
                T["h2d_all"].record(h2d)
                ready = q_ev
            step.enqueue(q_dev, out, lse, timers=timers, inputs_ready=ready)
            if d:
                for layer in range(L):
                    d2h.wait_event(step.out_ready[layer])
                    bs.copy_ptr(out_host.data_ptr() + layer * ob, out.data_ptr() + layer * ob, ob, stream=d2h)
                    bs.copy_ptr(lse_host.data_ptr() + layer * lb, lse.data_ptr() + layer * lb, lb, stream=d2h)
                cur.wait_stream(d2h)
            if h:
                cur.wait_stream(h2d)   # join the timer nodes recorded on the H2D stream
            T["end"].record(cur)
        one_t()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            one_t()
        for _ in range(5):
            g.replay()
            torch.cuda.synchronize()
        st = T["start"]
        r = {"total_ms": st.elapsed_time(T["end"]),
             "attn0_start_ms": st.elapsed_time(timers[0][0]),
             "attn_last_end_ms": st.elapsed_time(timers[L - 1][1]),
             "mig0_start_ms": st.elapsed_time(timers[0][2]),
             "attn_sum_ms": sum(t[0].elapsed_time(t[1]) for t in timers),
             "attn0_ms": timers[0][0].elapsed_time(timers[0][1]),
             "attn1_ms": timers[1][0].elapsed_time(timers[1][1])}
        if h:
            r["h2d0_done_ms"] = st.elapsed_time(T["h2d0"])
            r["h2d_all_done_ms"] = st.elapsed_time(T["h2d_all"])
        res[f"timeline_{name}"] = {k: round(v, 4) for k, v in r.items()}
        del g
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
