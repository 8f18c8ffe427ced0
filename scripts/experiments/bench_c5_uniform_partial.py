#!/usr/bin/env python
"""C5 (BASELINE.json configs[4]) at one GPU's share, timed on one B200.

    python scripts/bench_c5.py [--json out.json] [--gpus-share 8]

The 512-request burst (prompts log-uniform[128, 16k], Llama-3-8B shape, 32 layers, seed 0)
is spread over n GPUs (request i on GPU i mod n); this GPU takes requests i mod n == 0.
Every request's first half (prefix hit rate r = 0.5) sits in a global-store
pool (on another GPU in the paper's setting; here a second pool in this GPU's HBM, so the
copy is HBM-bound, not NVLink-bound).  One decode step of the burst = per layer: migrate
the layer's prefix blocks store -> home (H2, copy stream) and run split decode attention
over every request (H4, compute stream, gated on the layer's migration event, H3).
Reports: step time, attention-only and migration-only times, exposure
(T_step - T_attn) / T_attn, the migration's payload GB/s and the attention's HBM GB/s.
Graph-free, CUDA events, 3 warm-up + 10 timed steps; pools >> L2.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402


def run(gpus_share: int = 8, steps: int = 10, device=None) -> dict:
    """The C5 per-GPU burst step (module docstring); returns the result dict.  Also called
    by bench.py at N=1 (extra_configs.c5_share)."""
    args = argparse.Namespace(gpus_share=gpus_share, steps=steps)
    dev = device if device is not None else torch.device("cuda", 0)
    shape = synth.LLAMA3_8B
    g = torch.Generator().manual_seed(0)
    lo, hi = np.log(128.0), np.log(16384.0)
    lens_all = np.exp(lo + (hi - lo) * torch.rand(512, generator=g).numpy()).astype(np.int64)
    lens = lens_all[0::args.gpus_share]
    B, L = len(lens), shape.n_layers
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=61, device=dev)
    pt, bt = case.pools[0], case.block_tables[0]
    prefix = [int(x) for b in range(B) for x in bt[b, : synth.ceil_div(int(lens[b]), 16) // 2]]
    pidx = torch.tensor(prefix, dtype=torch.long, device=dev)
    store_t = pt.index_select(1, pidx).contiguous()
    home = bs.KVPool(L, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    store = bs.KVPool(L, store_t.shape[1], shape.hkv, shape.d, base=store_t.reshape(-1))
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32, device=dev)  # noqa: E731
    src_ids, dst_ids = i32(np.arange(len(prefix))), i32(prefix)
    sc = synth.default_scale(shape.d)
    btd, ksd = i32(bt), i32(ks)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(home, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    copy_s, comp_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event() for _ in range(L)]

    def step(mig=True, attn=True):
        for layer in range(L):
            if mig:
                with torch.cuda.stream(copy_s):
                    bs.kv_migrate_layer(store, home, layer, src_ids, dst_ids, stream=copy_s)
                    ev[layer].record(copy_s)
            if attn:
                with torch.cuda.stream(comp_s):
                    if mig:
                        comp_s.wait_event(ev[layer])
                    bs.split_decode_attention(home, layer, case.q[layer], btd, ksd, 0, sc, o, m, l,
                                              ws, stream=comp_s)

    def timed(**kw):
        for _ in range(3):
            step(**kw)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for s_ in (copy_s, comp_s):
            s_.wait_stream(cur)
        for _ in range(args.steps):
            step(**kw)
        for s_ in (copy_s, comp_s):
            cur.wait_stream(s_)
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    t_step = timed()
    t_attn = timed(mig=False)
    t_mig = timed(attn=False)
    tokens = int(lens.sum())
    mig_bytes = len(prefix) * home.chunk_bytes * L
    attn_bytes = tokens * 2 * shape.hkv * shape.d * 2 * L
    res = {"case": f"C5 one GPU's share of n={args.gpus_share}: {B} requests, {tokens} context tokens, "
                   f"{len(prefix)} prefix blocks per layer migrated (store pool in local HBM)",
           "step_ms": round(t_step, 4), "attn_only_ms": round(t_attn, 4), "mig_only_ms": round(t_mig, 4),
           "exposure": round((t_step - t_attn) / t_attn, 4),
           "mig_payload_GBps": round(mig_bytes / (t_mig * 1e-3) / 1e9, 1),
           "attn_kv_GBps": round(attn_bytes / (t_attn * 1e-3) / 1e9, 1),
           "mig_GB_per_step": round(mig_bytes / 1e9, 3), "attn_GB_per_step": round(attn_bytes / 1e9, 3),
           "decode_tokens_per_s": round(B / (t_step * 1e-3), 1)}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--gpus-share", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    res = run(a.gpus_share, a.steps)
    print(json.dumps(res), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
