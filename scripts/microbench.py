#!/usr/bin/env python
"""Per-kernel microbenchmarks (device time via CUDA events, warm, inputs > L2).

    python scripts/microbench.py [--only attn|mig] [--json out.json]

attention: one bs_split_decode_attention launch per iteration, one shard, shapes of the
BASELINE configs (C2 MHA, C3 GQA-4 long context, C4 GQA-8 mixed lengths); GB/s =
algorithmic bytes (KV + q + partials + block table) / event time.
migration: bs_kv_migrate_layer local copies (VEC16 vs BULK), payload GB/s (HBM traffic
is 2x).  Profiling hook: --ncu-attn / --ncu-mig run a few launches of one case only.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402


def attn_case(name, shape, lens, iters=20, warm=5, seed=1):
    dev = torch.device("cuda")
    lens = np.asarray(lens, dtype=np.int64)
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=seed, device=dev, layers=1)
    pt, bt = case.pools[0], case.block_tables[0]
    pool = bs.KVPool(1, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    B = len(lens)
    q = case.q[0]
    btd = torch.from_numpy(bt).to(dev)
    ksd = torch.from_numpy(ks).to(dev)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    sc = synth.default_scale(shape.d)
    for _ in range(warm):
        bs.split_decode_attention(pool, 0, q, btd, ksd, 0, sc, o, m, l, ws)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        bs.split_decode_attention(pool, 0, q, btd, ksd, 0, sc, o, m, l, ws)
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    med = t[len(t) // 2]
    kv = int(lens.sum()) * 2 * shape.hkv * shape.d * 2
    alg = kv + B * shape.hq * shape.d * 2 + B * shape.hq * (shape.d + 2) * 4 + 4 * int(
        sum(synth.ceil_div(int(x), 16) for x in lens))
    return {"case": name, "B": B, "G": shape.group, "tokens": int(lens.sum()), "us": round(med * 1e3, 2),
            "GBps": round(alg / (med * 1e-3) / 1e9, 1), "bytes": alg,
            "ws": ws.numel() > 16}


L2_BYTES = 126 * 2**20


def attn_case_graph(name, shape, lens, iters=40, seed=1, step_flags=False):
    """Device time of back-to-back launches without host overhead: ``iters`` launches are
    captured into one CUDA graph (per-launch time = replay time / iters), cycling over
    enough layers that the KV they read (>= 3x L2) cannot be served from L2.  Small
    problems (C3 B=1: 33 MB) are host-launch-bound under per-call event timing; this is
    the kernel's own latency as a graph-captured decode step would see it."""
    dev = torch.device("cuda")
    lens = np.asarray(lens, dtype=np.int64)
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    kv = int(lens.sum()) * 2 * shape.hkv * shape.d * 2
    nl = int(min(32, max(1, -(-3 * L2_BYTES // max(kv, 1)))))
    case = synth.device_shards(shape, lens, ks, seed=seed, device=dev, layers=nl)
    pt, bt = case.pools[0], case.block_tables[0]
    pool = bs.KVPool(nl, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    B = len(lens)
    btd = torch.from_numpy(bt).to(dev)
    ksd = torch.from_numpy(ks).to(dev)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    sc = synth.default_scale(shape.d)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x in range(nl):  # warm (also configures the kernel attributes outside capture)
            bs.split_decode_attention(pool, x, case.q[x], btd, ksd, 0, sc, o, m, l, ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    if step_flags:   # a decode step's layers: the fused local path, launches after the first
        ob = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)   # flagged
        wsl = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
            [pool], [bt.shape[1]], B, shape.hq)), dtype=torch.uint8, device=dev)
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            x = i % nl
            if step_flags:
                bs.split_decode_attention_local([pool], x, case.q[x], [btd], [0], ksd, sc, ob, l, wsl,
                                                stream=s, flags=bs.ATTN_PDL if i else 0)
            else:
                bs.split_decode_attention(pool, x, case.q[x], btd, ksd, 0, sc, o, m, l, ws, stream=s)
    info = bs.attention_last_launch()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / iters)
    med = sorted(ts)[len(ts) // 2]
    alg = kv + B * shape.hq * shape.d * 2 + B * shape.hq * (shape.d + 2) * 4 + 4 * int(
        sum(synth.ceil_div(int(x), 16) for x in lens))
    return {"case": name, "timing": "graph" + ("_step_flags" if step_flags else ""), "B": B,
            "G": shape.group, "tokens": int(lens.sum()), "launch": info,
            "layers_cycled": nl, "us": round(med * 1e3, 2),
            "GBps": round(alg / (med * 1e-3) / 1e9, 1), "bytes": alg}


def mig_case(name, shape, n_pairs, method, iters=20, warm=5):
    dev = torch.device("cuda")
    nb = n_pairs + 64
    src = bs.KVPool(1, nb, shape.hkv, shape.d)
    dst = bs.KVPool(1, nb, shape.hkv, shape.d)
    src.data.normal_()
    g = torch.Generator().manual_seed(0)
    s = torch.randperm(nb, generator=g)[:n_pairs].to(torch.int32).to(dev)
    d = torch.randperm(nb, generator=g)[:n_pairs].to(torch.int32).to(dev)
    for _ in range(warm):
        bs.kv_migrate_layer(src, dst, 0, s, d, method=method)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        bs.kv_migrate_layer(src, dst, 0, s, d, method=method)
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    med = t[len(t) // 2]
    by = n_pairs * src.chunk_bytes
    return {"case": name, "method": ["auto", "vec16", "bulk"][method], "pairs": n_pairs,
            "MiB": round(by / 2**20, 1), "us": round(med * 1e3, 2),
            "payload_GBps": round(by / (med * 1e-3) / 1e9, 1),
            "hbm_GBps": round(2 * by / (med * 1e-3) / 1e9, 1)}


def mig_extra_cases(args, iters=20, warm=5):
    """NEXT F2 (head pages) and F3 (multi-layer, one launch) copies, payload GB/s."""
    dev = torch.device("cuda")
    out = []

    def timeit(fn):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters

    shape = synth.LLAMA3_8B
    n = 4096
    src = bs.KVPool(8, n + 64, 8, 128)
    dst = bs.KVPool(8, n + 64, 8, 128)
    cold = bs.KVPool(8, n + 64, 2, 128)
    g = torch.Generator().manual_seed(0)
    s = torch.randperm(n + 64, generator=g)[:n].to(torch.int32).to(dev)
    d = torch.randperm(n + 64, generator=g)[:n].to(torch.int32).to(dev)
    ms = timeit(lambda: bs.kv_migrate_heads_layer(src, cold, 0, s, d, 6, 0, 2))
    by = n * 2 * 2 * 16 * 128 * 2
    out.append({"case": "F2_heads_2of8_4096blocks", "us": round(ms * 1e3, 2),
                "payload_GBps": round(by / (ms * 1e-3) / 1e9, 1), "MiB": by / 2**20})
    ms = timeit(lambda: bs.kv_migrate_layers(src, dst, 0, 8, s, d))
    by = 8 * n * src.chunk_bytes
    out.append({"case": "F3_8layers_4096chunks_one_launch", "us": round(ms * 1e3, 2),
                "payload_GBps": round(by / (ms * 1e-3) / 1e9, 1), "MiB": by / 2**20})
    ms = timeit(lambda: [bs.kv_migrate_layer(src, dst, x, s, d) for x in range(8)])
    out.append({"case": "F3_8layers_4096chunks_per_layer_launches", "us": round(ms * 1e3, 2),
                "payload_GBps": round(by / (ms * 1e-3) / 1e9, 1), "MiB": by / 2**20})
    for r in out:
        print(json.dumps(r), flush=True)
    return out


def tasks_cases(iters=20, warm=5):
    """Cost of the fused cross-GPU exchange epilogue on one GPU: two C2 problems (B=64 x
    2048, 2 shards each, 4 GiB of KV) as (i) two single-GPU fused launches, (ii) two
    task launches each mixing a shard of both problems (the N=2 ring's launch shape) with
    gpu-scope counters, (iii) the same with system-scope counters + done counters."""
    dev = torch.device("cuda")
    shape = synth.LLAMA2_7B
    lens = np.full(64, 2048)
    ks = synth.block_aligned_split(lens, 2)
    probs = []
    for seed in (1, 2):
        case = synth.device_shards(shape, lens, ks, seed=seed, device=dev, layers=1)
        pools = [bs.KVPool(1, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1)) for pt in case.pools]
        bts = [torch.from_numpy(bt).to(dev) for bt in case.block_tables]
        mb = [t.shape[1] for t in bts]
        n = bs.attention_problem_workspace_size(64, shape.hq, shape.hkv, shape.d, mb)
        probs.append({"pools": pools, "bts": bts, "q": case.q[0], "ks": torch.from_numpy(ks).to(dev),
                      "mb": mb, "ws": torch.zeros(max(n, 256), dtype=torch.uint8, device=dev),
                      "out": torch.empty(64, shape.hq, shape.d, dtype=torch.bfloat16, device=dev),
                      "lse": torch.empty(64, shape.hq, device=dev),
                      "done": torch.zeros(1, dtype=torch.int32, device=dev)})
    sc = synth.default_scale(shape.d)
    kv = int(lens.sum()) * 2 * shape.hkv * shape.d * 2 * 2

    def desc(P, cross):
        return {"q": P["q"], "kv_split": P["ks"], "max_blocks": P["mb"], "out": P["out"],
                "lse": P["lse"], "workspace": P["ws"], "done": P["done"] if cross else None,
                "cross_device": cross}

    def local():
        for P in probs:
            bs.split_decode_attention_local(P["pools"], 0, P["q"], P["bts"], [0, 1], P["ks"], sc,
                                            P["out"], P["lse"], P["ws"])

    def tasks(cross):
        A, B = probs
        d = [desc(A, cross), desc(B, cross)]
        bs.split_decode_attention_tasks(d, [(A["pools"][0], A["bts"][0], 0, 0),
                                            (B["pools"][1], B["bts"][1], 1, 1)], 0, 64, shape.hq, sc)
        bs.split_decode_attention_tasks(d, [(A["pools"][1], A["bts"][1], 1, 0),
                                            (B["pools"][0], B["bts"][0], 0, 1)], 0, 64, shape.hq, sc)
    out = []
    for name, fn in (("two_local_fused_launches", local), ("two_task_launches_gpu_scope",
                                                             lambda: tasks(False)),
                     ("two_task_launches_sys_scope_done", lambda: tasks(True))):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / iters
        r = {"case": "tasks_C2x2_" + name, "us": round(ms * 1e3, 2),
             "kv_GBps": round(kv / (ms * 1e-3) / 1e9, 1)}
        print(json.dumps(r), flush=True)
        out.append(r)
    return out


def append_cases(iters=200, warm=20):
    """H7 append (bs_kv_append_token): one launch per layer writing each request's new
    K/V rows; per-call time graph-timed (40 captured launches) and per-call event-timed."""
    dev = torch.device("cuda")
    out = []
    for name, shape, B in (("C2_B64", synth.LLAMA2_7B, 64), ("C3_B8", synth.LLAMA3_8B, 8),
                           ("C4_B256", synth.LLAMA2_70B, 256)):
        nb = B * 4
        pool = bs.KVPool(1, nb, shape.hkv, shape.d)
        bt = torch.arange(nb, dtype=torch.int32, device=dev).view(B, 4)
        pos = torch.randint(0, 64, (B,), dtype=torch.int32, device=dev)
        k = torch.randn(B, shape.hkv, shape.d, device=dev).to(torch.bfloat16)
        v = torch.randn(B, shape.hkv, shape.d, device=dev).to(torch.bfloat16)
        fn = lambda: bs.kv_append_token(pool, 0, k, v, bt, pos)  # noqa: E731
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(40):
                    fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters // 40):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (iters // 40 * 40)
        by = 2 * B * 2 * shape.hkv * shape.d * 2   # rows read + written
        r = {"case": f"append_{name}", "B": B, "hkv": shape.hkv, "us_graph": round(us, 2),
             "bytes": by, "GBps": round(by / (us * 1e-6) / 1e9, 1)}
        print(json.dumps(r), flush=True)
        out.append(r)
    return out


def push_view_cases(iters=20, warm=5):
    """The P2P push kernel's own rate: bs_kv_migrate_layer into a remote view (a pool
    handle whose desc.device is another ordinal) runs on one CTA per SM; emulated over
    local memory, so this is the issue rate of the capped grid (HBM-bound here), to be
    compared with NVLink's 900 GB/s per direction the real push is bounded by."""
    dev = torch.device("cuda")
    out = []
    for name, shape, n in (("C2_handoff_384x256KiB", synth.LLAMA2_7B, 384),
                           ("C4_handoff_512x64KiB", synth.LLAMA3_8B, 512),
                           ("C2_bulk_8192x256KiB", synth.LLAMA2_7B, 8192)):
        nb = n + 64
        src = bs.KVPool(1, nb, shape.hkv, shape.d)
        dst = bs.KVPool(1, nb, shape.hkv, shape.d)
        view = bs.pool_view(1, nb, shape.hkv, shape.d, dst.data.data_ptr(),
                            torch.cuda.current_device() + 1)
        g = torch.Generator().manual_seed(0)
        s_ = torch.randperm(nb, generator=g)[:n].to(torch.int32).to(dev)
        d_ = torch.randperm(nb, generator=g)[:n].to(torch.int32).to(dev)
        for kind, target in (("remote_view_1cta_per_sm", view), ("local_full_grid", dst)):
            fn = lambda: bs.kv_migrate_layer(src, target, 0, s_, d_)  # noqa: E731
            for _ in range(warm):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / iters
            by = n * src.chunk_bytes
            r = {"case": f"{name}_{kind}", "us": round(us, 2), "payload_GBps": round(by / (us * 1e-6) / 1e9, 1),
                 "vs_nvlink_900": round(by / (us * 1e-6) / 1e9 / 900.0, 2)}
            print(json.dumps(r), flush=True)
            out.append(r)
        del src, dst
        torch.cuda.empty_cache()
    return out


RAGGED_EXTRA_BPS = []


def ragged_cases(iters=20, warm=5, step_flags=False):
    """Mixed-length shards through the single-GPU fused launch: uniform grid (max_blocks-
    wide ranges) vs the ragged plan (bs_attention_ragged_plan).  GB/s = algorithmic bytes
    (KV + q + bf16 O + lse + block table) / time."""
    dev = torch.device("cuda")
    out = []
    cases = {
        "C4_gqa8_mixed_B256": (synth.LLAMA2_70B, synth.mixed_lengths(256, seed=0) // 8),
        "C4_gqa8_mixed_B256_seed3": (synth.LLAMA2_70B, synth.mixed_lengths(256, seed=3) // 8),
        "C2_mha_B64_2048": (synth.LLAMA2_7B, np.full(64, 2048)),
        "C3_gqa4_B8_8192": (synth.LLAMA3_8B, np.full(8, 8192)),
    }
    for name, (shape, lens) in cases.items():
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
        wsu = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
            [pool], [bts[0].shape[1]], B, shape.hq)), dtype=torch.uint8, device=dev)
        plans = {}
        variants = [("ragged", 0, "1"), ("ragged_reqorder", 0, "0"), ("ragged_bps64", 64, "1"),
                    ("ragged_bps32", 32, "1")]
        variants += [(f"ragged_bps{x}", x, "1") for x in RAGGED_EXTRA_BPS]
        for kind, bps, order in variants:
            os.environ["BS_RAGGED_ORDER"] = order
            pl = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d,
                                          max_blocks_per_range=bps).to(dev)
            plans[kind] = (pl, torch.zeros(max(16, pl.workspace_bytes), dtype=torch.uint8, device=dev))
        os.environ.pop("BS_RAGGED_ORDER")
        alg = int(lens.sum()) * 2 * shape.hkv * shape.d * 2 + B * shape.hq * shape.d * 2 + \
            B * shape.hq * (shape.d * 2 + 4) + 4 * int(sum(synth.ceil_div(int(x), 16) for x in lens))
        fns = {"uniform": (None, lambda: bs.split_decode_attention_local([pool], 0, case.q[0], bts, [0],
                                                                         ksd, sc, o, lse, wsu))}
        for kind, (pl, wsr) in plans.items():
            fns[kind] = (pl, lambda pl=pl, wsr=wsr: bs.split_decode_attention_local_ragged(
                [pool], 0, case.q[0], bts, [0], ksd, sc, pl, o, lse, wsr))
        if step_flags:   # 20 launches per graph, the PDL flag on all but the first
            for kind in list(fns):
                pl, wsr = plans[kind] if kind in plans else (None, wsu)

                def launch(flags, pl=pl, wsr=wsr):
                    if pl is None:
                        bs.split_decode_attention_local([pool], 0, case.q[0], bts, [0], ksd, sc, o, lse,
                                                        wsu, flags=flags)
                    else:
                        bs.split_decode_attention_local_ragged([pool], 0, case.q[0], bts, [0], ksd, sc, pl,
                                                               o, lse, wsr, flags=flags)
                launch(0)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                st = torch.cuda.Stream()
                with torch.cuda.graph(g, stream=st):
                    for i in range(20):
                        launch(bs.ATTN_PDL if i else 0)
                fns[kind] = (pl, lambda g=g: g.replay(), 20)
        for kind, item in fns.items():
            plan, fn = item[0], item[1]
            per = item[2] if len(item) > 2 else 1
            for _ in range(warm):
                fn()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(iters)]
            for a, b in evs:
                a.record()
                fn()
                b.record()
            torch.cuda.synchronize()
            t = sorted(a.elapsed_time(b) / per for a, b in evs)
            med = t[len(t) // 2]
            r = {"case": f"{name}_{kind}", "timing": "graph_step_flags" if step_flags else "event",
                 "B": B, "G": shape.group, "tokens": int(lens.sum()),
                 "us": round(med * 1e3, 2), "GBps": round(alg / (med * 1e-3) / 1e9, 1), "bytes": alg,
                 "items": plan.n_work if plan is not None else None,
                 "max_parts": plan.max_parts if plan is not None else None}
            print(json.dumps(r), flush=True)
            out.append(r)
        del case, pool
        torch.cuda.empty_cache()
    return out


ATTN = {
    "C2_mha_B64_2048": (synth.LLAMA2_7B, [2048] * 64),
    "C2_shard_B64_1024": (synth.LLAMA2_7B, [1024] * 64),
    "C3_gqa4_B8_8192": (synth.LLAMA3_8B, [8192] * 8),
    "C3_gqa4_B1_8192": (synth.LLAMA3_8B, [8192] * 1),
    "C3_gqa4_B32_8192": (synth.LLAMA3_8B, [8192] * 32),
    "C3_gqa4_B8_32768_1gpu": (synth.LLAMA3_8B, [32768] * 8),
    "C4_gqa8_mixed_B256": (synth.LLAMA2_70B, list(synth.mixed_lengths(256, seed=0) // 8)),
}
# diagnostics: same KV bytes, different group size / kv-head count (--diag)
DIAG = {
    "D_hkv8_G1_B256_2048": (synth.Shape(1, 8, 8, 128), [2048] * 256),
    "D_hkv8_G4_B256_2048": (synth.Shape(1, 32, 8, 128), [2048] * 256),
    "D_hkv8_G8_B256_2048": (synth.Shape(1, 64, 8, 128), [2048] * 256),
    "D_hkv32_G1_B64_2048": (synth.Shape(1, 32, 32, 128), [2048] * 64),
    "D_hkv32_G2_B64_2048": (synth.Shape(1, 64, 32, 128), [2048] * 64),
    "D_hkv8_G8_B256_684": (synth.Shape(1, 64, 8, 128), [684] * 256),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["attn", "mig", "tasks", "ragged", "append", "push"])
    ap.add_argument("--case")
    ap.add_argument("--json")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--diag", action="store_true", help="group-size / kv-head diagnostics")
    ap.add_argument("--ragged-bps", type=int, action="append", default=[],
                    help="extra ragged-plan range lengths to time")
    ap.add_argument("--graph", action="store_true",
                    help="attention: time graph-captured back-to-back launches over >= 3x L2 of KV")
    ap.add_argument("--step-flags", action="store_true",
                    help="--graph through the fused local path with the BS_ATTN_PDL flag on every "
                         "launch after the first (the production policy of a decode step)")
    ap.add_argument("--seeds", type=int, default=1,
                    help="repeat every attention case over seeds 0..n-1 (block placement and "
                         "values; C4 also its lengths) and report mean / spread")
    args = ap.parse_args()
    res = []
    if args.only in (None, "attn"):
        for name, (shape, lens) in (DIAG if args.diag else ATTN).items():
            if args.case and args.case != name:
                continue
            if args.graph:
                r = attn_case_graph(name, shape, lens, step_flags=args.step_flags)
            elif args.seeds <= 1:
                r = attn_case(name, shape, lens, iters=args.iters)
            else:
                runs = []
                for sd in range(args.seeds):
                    ln = (synth.mixed_lengths(256, seed=sd) // 8) if name.startswith("C4") else lens
                    runs.append(attn_case(name, shape, ln, iters=args.iters, seed=sd))
                g = [x["GBps"] for x in runs]
                r = {"case": name, "seeds": args.seeds, "GBps_mean": round(float(np.mean(g)), 1),
                     "GBps_min": min(g), "GBps_max": max(g),
                     "us_mean": round(float(np.mean([x["us"] for x in runs])), 2)}
            print(json.dumps(r), flush=True)
            res.append(r)
    if args.only in (None, "mig"):
        for name, shape, n in (("C2_chunk256K_384", synth.LLAMA2_7B, 384),
                               ("C2_chunk256K_8192", synth.LLAMA2_7B, 8192),
                               ("C4_chunk64K_512", synth.LLAMA3_8B, 512),
                               ("C4_chunk64K_8192", synth.LLAMA3_8B, 8192)):
            if args.case and args.case != name:
                continue
            for method in (1, 2):
                r = mig_case(name, shape, n, method, iters=args.iters)
                print(json.dumps(r), flush=True)
                res.append(r)
    if args.only in (None, "mig"):
        res += mig_extra_cases(args)
    if args.only in (None, "tasks"):
        res += tasks_cases(iters=args.iters)
    if args.only in (None, "append"):
        res += append_cases()
    if args.only in (None, "push"):
        res += push_view_cases()
    if args.only in (None, "ragged"):
        RAGGED_EXTRA_BPS.extend(args.ragged_bps)
        res += ragged_cases(iters=args.iters, step_flags=args.step_flags)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
