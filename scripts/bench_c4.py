#!/usr/bin/env python
"""C4 (BASELINE.json configs[3]) at one GPU's share, timed on one B200.

    python scripts/bench_c4.py [--json out.json] [--seed 0]

Llama-2-70B shape (80 layers, 64 q / 8 kv heads, d 128), B = 256 mixed prompt /
generation lengths (Fig. 7 recipe), every request split 8-way
block-aligned across 8 GPUs; this GPU holds shard 3 of every request (all 80 layers
resident, ~58 GB) and receives 8192 tokens of layer-wise migrated KV per step (512 chunks
of 64 KiB per layer, from a second pool standing in for the sending GPU: HBM-bound here,
NVLink-bound at 8 GPUs).  One step = per layer: the hand-off copy (copy stream) and the
ragged-plan attention over the shard (compute stream, gated on that layer's copy event).
Reports step / attention-only / migration-only times, exposure, GB/s.
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


def run(seed: int = 0, steps: int = 10, handoff_tokens: int = 8192, device=None) -> dict:
    """The C4 per-GPU step (module docstring); returns the result dict.  Also called by
    bench.py at N=1 (extra_configs.c4_share)."""
    args = argparse.Namespace(seed=seed, steps=steps, handoff_tokens=handoff_tokens)
    dev = device if device is not None else torch.device("cuda", 0)
    shape = synth.LLAMA2_70B
    L = shape.n_layers
    lens = synth.mixed_lengths(256, seed=args.seed)
    ks8 = synth.block_aligned_split(lens, 8)
    shard = (ks8[:, 4] - ks8[:, 3]).astype(np.int64)
    ks = np.stack([np.zeros_like(shard), shard], 1).astype(np.int32)
    n_hand = args.handoff_tokens // 16
    case = synth.device_shards(shape, shard, ks, seed=53, device=dev, spare_blocks=n_hand)
    pt, bt = case.pools[0], case.block_tables[0]
    B = len(lens)
    pool = bs.KVPool(L, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    used = {int(x) for x in bt.ravel() if x >= 0}
    free = [i for i in range(pt.shape[1]) if i not in used][:n_hand]
    sender = bs.KVPool(L, n_hand, shape.hkv, shape.d)
    sender.data.normal_()
    i32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32, device=dev)  # noqa: E731
    src_ids, dst_ids = i32(np.arange(n_hand)), i32(free)
    sc = synth.default_scale(shape.d)
    plan = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d, pack_short=True).to(dev)
    ws = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device=dev)
    btd, ksd = i32(bt), i32(ks)
    out = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, shape.hq, device=dev)
    copy_s, comp_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event() for _ in range(L)]

    def step(mig=True, attn=True):
        for layer in range(L):
            if mig:
                with torch.cuda.stream(copy_s):
                    bs.kv_migrate_layer(sender, pool, layer, src_ids, dst_ids, stream=copy_s)
                    ev[layer].record(copy_s)
            if attn:
                with torch.cuda.stream(comp_s):
                    if mig:
                        comp_s.wait_event(ev[layer])
                    # layers > 0: programmatic dependents of the previous layer's launch
                    # (the hand-off writes are joined by the event, not stream order)
                    bs.split_decode_attention_local_ragged([pool], layer, case.q[layer], [btd], [0], ksd,
                                                           sc, plan, out, lse, ws, stream=comp_s,
                                                           flags=bs.ATTN_PDL if layer else 0)

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
    tokens = int(shard.sum())
    mig_bytes = n_hand * pool.chunk_bytes * L
    attn_bytes = tokens * 2 * shape.hkv * shape.d * 2 * L
    res = {"case": f"C4 one GPU's shard (3 of 8), seed {args.seed}: {B} requests, {tokens} shard tokens, "
                   f"{L} layers; {args.handoff_tokens} tokens handed off per layer",
           "step_ms": round(t_step, 4), "attn_only_ms": round(t_attn, 4), "mig_only_ms": round(t_mig, 4),
           "exposure": round((t_step - t_attn) / t_attn, 4),
           "mig_payload_GBps": round(mig_bytes / (t_mig * 1e-3) / 1e9, 1),
           "attn_kv_GBps": round(attn_bytes / (t_attn * 1e-3) / 1e9, 1),
           "hbm_floor_exposure": round(2 * mig_bytes / attn_bytes, 4),
           "decode_tokens_per_s_per_gpu_share": round(B / (t_step * 1e-3), 1)}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--handoff-tokens", type=int, default=8192)
    a = ap.parse_args()
    res = run(a.seed, a.steps, a.handoff_tokens)
    print(json.dumps(res), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
