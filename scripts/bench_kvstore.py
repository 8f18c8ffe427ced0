#!/usr/bin/env python
"""NEXT row F1 measurement: Global KV Cache Store CPU tier on one B200.

    python scripts/bench_kvstore.py [--json out.json]

Workload = the paper's worked example (eqs. 14-17): Llama-3.1-8B
shape (32 layers, 8 KV heads, d=128 -> S_kv = 4096 B/token/layer), prompts of L = 1000
tokens, prefix hit rate r = 0.5.  Per layer the store fetches the 500-token prefix
(HtoD) of R arriving requests and stores their 500 incremental tokens (DtoH), while the
GPU computes split decode attention over a resident batch (32 x 8192 tokens, GQA-4).
Reports fetch / store GB/s alone, compute alone, the pipelined total, exposure =
(T_total - T_compute)/T_compute, and the eq. 13 prediction at the measured bandwidth.
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
from paper_2510_13223_b200.kvstore import KVStore, ThreeStagePipeline, transfer_model  # noqa: E402


def timed(fn, iters=10, warm=3):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=4)
    ap.add_argument("--engine", choices=["staged", "ce", "sm"], default="staged")
    ap.add_argument("--json")
    args = ap.parse_args()
    dev = torch.device("cuda")
    shape = synth.LLAMA3_8B
    L = shape.n_layers
    R = args.requests
    prefix_blocks = synth.ceil_div(500, 16)            # r * L tokens per request
    nf = R * prefix_blocks
    # resident batch for the compute stage
    B, S = 32, 8192
    lens = np.full(B, S)
    ks = np.stack([np.zeros(B), lens], 1).astype(np.int32)
    pool_t, bt = synth.device_pool(shape, lens, seed=3, device=dev, spare_blocks=2 * nf, layers=L)
    pool = bs.KVPool(L, pool_t.shape[1], shape.hkv, shape.d, base=pool_t.reshape(-1))
    used = set(int(x) for x in bt.ravel() if x >= 0)
    free = [i for i in range(pool.num_blocks) if i not in used]
    store = KVStore(L, 2 * nf, shape.hkv, shape.d)
    store.pool.data.view(torch.int16).random_()
    i32 = lambda x: torch.as_tensor(np.asarray(x, dtype=np.int32)).to(dev)
    conv = i32 if args.engine == "sm" else list
    f_store, f_dev = conv(list(range(nf))), conv(free[:nf])
    s_dev, s_store = conv(free[nf:2 * nf]), conv(list(range(nf, 2 * nf)))
    eng = args.engine
    q = synth.device_q(shape, B, 1, dev, L)
    btd, ksd = i32(bt), i32(ks)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    sc = synth.default_scale(shape.d)

    def compute(layer):
        bs.split_decode_attention(pool, layer, q[layer], btd, ksd, 0, sc, o, m, l, ws)

    side = torch.cuda.Stream()

    def on_side(fn):
        def run():
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                fn()
            torch.cuda.current_stream().wait_stream(side)
        return run

    if eng == "staged":
        fsp, ssp = store.prepare(pool, f_store, f_dev), store.prepare(pool, s_store, s_dev)
        t_fetch = timed(on_side(lambda: [store.fetch_staged(pool, x, fsp) for x in range(L)])) / L
        t_store = timed(on_side(lambda: [store.store_staged(pool, x, ssp) for x in range(L)])) / L
    else:
        t_fetch = timed(on_side(lambda: [store.fetch_layer(pool, x, f_store, f_dev, engine=eng)
                                         for x in range(L)])) / L
        t_store = timed(on_side(lambda: [store.store_layer(pool, x, s_dev, s_store, engine=eng)
                                         for x in range(L)])) / L
    t_comp = timed(lambda: [compute(x) for x in range(L)]) / L
    pipe = ThreeStagePipeline(store, pool, L, compute, fetch_pairs=(f_store, f_dev),
                              store_pairs=(s_dev, s_store), engine=eng)
    t_total = timed(lambda: pipe.enqueue()) / L
    nbytes = nf * pool.chunk_bytes
    bw_f = nbytes / (t_fetch * 1e-3)
    s_kv = shape.kv_bytes_per_token_layer
    _, t_kv_pred = transfer_model(s_kv, 1000 * R, 0.5, bw_f, 0.27, L)
    res = {
        "engine": eng,
        "workload": f"Llama-3.1-8B shape, {R} requests x L=1000 tokens, r=0.5 -> {nf} chunks "
                    f"({nbytes / 2**20:.1f} MiB) fetched + stored per layer; compute = split decode "
                    f"attention B={B} x {S} (GQA-4)",
        "fetch_ms_per_layer": round(t_fetch, 4), "fetch_GBps": round(bw_f / 1e9, 2),
        "store_ms_per_layer": round(t_store, 4), "store_GBps": round(nbytes / (t_store * 1e-3) / 1e9, 2),
        "compute_ms_per_layer": round(t_comp, 4),
        "pipelined_ms_per_layer": round(t_total, 4),
        "serial_ms_per_layer": round(t_fetch + t_comp + t_store, 4),
        "exposure": round((t_total - t_comp) / t_comp, 4),
        "eq13_T_KV_ms_at_measured_B": round(t_kv_pred * 1e3, 4),
    }
    print(json.dumps(res), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
