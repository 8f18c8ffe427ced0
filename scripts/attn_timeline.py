#!/usr/bin/env python
"""Per-CTA timeline of one attention launch (diagnostics; needs the BS_TIMELINE build).

    BS_TIMELINE=1 python scripts/attn_timeline.py [--case C3_gqa4_B1_8192] [--json out.json]

The timeline build (`build(timeline=True)`, libbanaserve_timeline.so) stamps %globaltimer
in every CTA of the tensor-core kernel: entry, first K/V stage landed (warp 0), all loops
done, arrival counter resolved, exit.  L2 is flushed (256 MiB write) before the timed
launch, so every K/V byte comes from HBM.  Output: quantiles (us, relative to the first
CTA's entry) of each stamp and of the phases between them, split by last-arriver.
"""
import argparse
import ctypes
import json
import os
import sys

os.environ["BS_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import paper_2510_13223_b200 as bs  # noqa: E402
import synth  # noqa: E402
from microbench import ATTN  # noqa: E402

KT = 16384
KC = 8   # stamp columns (see attention.cu: [6] = griddepcontrol.wait returned)


def q(x, ps=(0, 10, 50, 90, 100)):
    x = np.asarray(x, dtype=np.float64)
    return {f"p{p}": round(float(np.percentile(x, p)), 2) for p in ps} if len(x) else {}


def run(name, reps=5, ragged_bps=None):
    shape, lens = ATTN[name]
    dev = torch.device("cuda")
    lens = np.asarray(lens, dtype=np.int64)
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=1, device=dev, layers=1)
    pt, bt = case.pools[0], case.block_tables[0]
    pool = bs.KVPool(1, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    B = len(lens)
    btd = torch.from_numpy(bt).to(dev)
    ksd = torch.from_numpy(ks).to(dev)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    sc = synth.default_scale(shape.d)
    call = lambda: bs.split_decode_attention(pool, 0, case.q[0], btd, ksd, 0, sc, o, m, l, ws)  # noqa: E731
    if ragged_bps is not None:  # fused local path over a ragged plan (longest range first)
        plan = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d,
                                        max_blocks_per_range=ragged_bps).to(dev)
        wsr = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device=dev)
        ob = torch.empty(B, shape.hq, shape.d, dtype=torch.bfloat16, device=dev)
        call = lambda: bs.split_decode_attention_local_ragged([pool], 0, case.q[0], [btd], [0], ksd, sc,  # noqa: E731
                                                              plan, ob, l, wsr)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    L = bs.lib()
    L.bs_timeline_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    L.bs_timeline_read.restype = ctypes.c_int32
    out = []
    for _ in range(reps):
        call()
        flush.fill_(1)
        torch.cuda.synchronize()
        assert L.bs_timeline_reset() == 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        buf = np.zeros((KT, KC), dtype=np.uint64)
        assert L.bs_timeline_read(buf.ctypes.data, buf.nbytes) == 0
        out.append((a.elapsed_time(b) * 1e3, buf))
    ev_us, buf = sorted(out, key=lambda x: x[0])[len(out) // 2]
    nz = buf[:, 4] > 0
    t = buf[nz].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t[:, :5] - t0) / 1e3
    last = ((t[:, 5] >> 16) & 1).astype(bool)
    has3 = t[:, 3] > 0     # CTAs that took part in a split-K arrival
    has1 = t[:, 1] > 0
    res = {
        "case": name + ("" if ragged_bps is None else f"_ragged_bps{ragged_bps}"),
        "ctas": int(nz.sum()), "event_us": round(ev_us, 2),
        "span_us": round(float(rel[:, 4].max()), 2),
        "entry": q(rel[:, 0]),
        "first_data_after_entry": q((rel[:, 1] - rel[:, 0])[has1]),
        "loop_done_after_entry": q(rel[:, 2] - rel[:, 0]),
        "loop_done": q(rel[:, 2]),
        "arrival_after_loop": q((rel[:, 3] - rel[:, 2])[has3]),
        "merge_last_arriver": q((rel[:, 4] - rel[:, 3])[last & has3]),
        "epilogue_single_range": q((rel[:, 4] - rel[:, 2])[~has3]),
        "exit_last_arriver": q(rel[last, 4]),
        "exit_others": q(rel[~last, 4]),
        "sms_used": int(len(np.unique(t[:, 5] & 0xFFFF))),
    }
    # per-SM load: loop duration grouped by how many CTAs of the launch ran on the same SM
    sm = (t[:, 5] & 0xFFFF).astype(np.int64)
    per_sm = np.bincount(sm, minlength=int(sm.max()) + 1)[sm]
    loop = rel[:, 2] - rel[:, 0]
    nbk = (t[:, 5] >> 20).astype(np.int64)
    res["max_blocks_per_cta"] = int(nbk.max())
    res["loop_us_per_block_by_size"] = {}
    for lo, hi in ((1, 16), (16, 64), (64, 128), (128, 256), (256, 513)):
        sel = (nbk >= lo) & (nbk < hi)
        if sel.any():
            res["loop_us_per_block_by_size"][f"{lo}-{hi - 1}"] = dict(
                n=int(sel.sum()), loop_us=q(loop[sel]), start_us=q(rel[sel, 0]))
    res["loop_by_ctas_on_sm"] = {int(c): dict(n=int((per_sm == c).sum()), **q(loop[per_sm == c]))
                                 for c in np.unique(per_sm)}
    # where the spread comes from: loop time by SM-id quarter (the two dies are expected
    # to split the id range), by grid position, and whether the same SMs are slow in every
    # repetition (correlation of per-SM mean loop time between repetitions)
    nsm = int(sm.max()) + 1
    res["loop_by_sm_quarter"] = {f"{k * nsm // 4}-{(k + 1) * nsm // 4 - 1}": q(
        loop[(sm >= k * nsm // 4) & (sm < (k + 1) * nsm // 4)]) for k in range(4)}
    lin = np.nonzero(nz)[0]
    res["loop_by_grid_quarter"] = {f"q{k}": q(loop[(lin >= k * len(lin) // 4) & (lin < (k + 1) * len(lin) // 4)])
                                   for k in range(4)}

    def per_sm_mean(b):
        m = b[:, 4] > 0
        tt = b[m].astype(np.int64)
        s_ = (tt[:, 5] & 0xFFFF).astype(np.int64)
        lp = (tt[:, 2] - tt[:, 0]) / 1e3
        cnt = np.bincount(s_, minlength=nsm)
        tot = np.bincount(s_, weights=lp, minlength=nsm)
        return np.where(cnt > 0, tot / np.maximum(cnt, 1), np.nan)
    means = [per_sm_mean(b) for _, b in out]
    cors = []
    for i in range(len(means)):
        for j in range(i + 1, len(means)):
            ok = ~np.isnan(means[i]) & ~np.isnan(means[j])
            if ok.sum() > 2:
                cors.append(float(np.corrcoef(means[i][ok], means[j][ok])[0, 1]))
    res["per_sm_loop_correlation_across_reps"] = q(cors) if cors else {}
    return res


def pdl_pair(name, reps=5, graph=False):
    """Two launches of one case back to back on one stream (the second reading the next
    layer's KV), L2 flushed before: per-CTA stamps of both (rows of launch 2 start at
    KT / 2).  Run once with BS_ATTN_PDL=1 and once with 0 to see whether the second grid's
    CTAs become resident, prefetch and wait while the first drains."""
    shape, lens = ATTN[name]
    dev = torch.device("cuda")
    lens = np.asarray(lens, dtype=np.int64)
    ks = np.stack([np.zeros_like(lens), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=1, device=dev, layers=2)
    pt, bt = case.pools[0], case.block_tables[0]
    pool = bs.KVPool(2, pt.shape[1], shape.hkv, shape.d, base=pt.reshape(-1))
    B = len(lens)
    btd = torch.from_numpy(bt).to(dev)
    ksd = torch.from_numpy(ks).to(dev)
    o = torch.empty(B, shape.hq, shape.d, device=dev)
    m = torch.empty(B, shape.hq, device=dev)
    l = torch.empty(B, shape.hq, device=dev)
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, B, shape.hq, bt.shape[1])),
                     dtype=torch.uint8, device=dev)
    sc = synth.default_scale(shape.d)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    L = bs.lib()
    L.bs_timeline_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    L.bs_timeline_read.restype = ctypes.c_int32
    spans = []
    g = None
    if graph:  # both launches captured in one CUDA graph: no host gap between them
        for layer in (0, 1):
            bs.split_decode_attention(pool, layer, case.q[layer], btd, ksd, 0, sc, o, m, l, ws)
        torch.cuda.synchronize()
        s_ = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s_):
            for layer in (0, 1):
                bs.split_decode_attention(pool, layer, case.q[layer], btd, ksd, 0, sc, o, m, l, ws)
    for _ in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        assert L.bs_timeline_reset() == 0
        if g is not None:
            g.replay()   # the captured launches keep the rows they were captured with
        else:
            for layer in (0, 1):
                bs.split_decode_attention(pool, layer, case.q[layer], btd, ksd, 0, sc, o, m, l, ws)
        info = bs.attention_last_launch()
        torch.cuda.synchronize()
        buf = np.zeros((KT, KC), dtype=np.uint64)
        assert L.bs_timeline_read(buf.ctypes.data, buf.nbytes) == 0
        a, b2 = buf[: KT // 2], buf[KT // 2:]
        a = a[a[:, 4] > 0].astype(np.int64)
        b2 = b2[b2[:, 4] > 0].astype(np.int64)
        t0 = a[:, 0].min()
        rel = lambda x: (x - t0) / 1e3  # noqa: E731
        r = {"case": name, "pdl": info["pdl"], "cluster": info["cluster"], "ranges": info["ranges"],
             "ctas": [int(len(a)), int(len(b2))],
             "A_exit": q(rel(a[:, 4])), "B_entry": q(rel(b2[:, 0])),
             "B_wait_return": q(rel(b2[:, 6][b2[:, 6] > 0])) if (b2[:, 6] > 0).any() else {},
             "B_first_data": q(rel(b2[:, 1][b2[:, 1] > 0])), "B_loop_done": q(rel(b2[:, 2])),
             "B_exit": q(rel(b2[:, 4])), "pair_span_us": round(float(rel(b2[:, 4]).max()), 2),
             "graph": graph}
        spans.append(r)
    spans.sort(key=lambda r: r["pair_span_us"])
    return spans[len(spans) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append")
    ap.add_argument("--json")
    ap.add_argument("--pdl-pair", action="store_true",
                    help="two back-to-back launches per case (set BS_ATTN_PDL=0/1 outside)")
    ap.add_argument("--ragged-bps", type=int, action="append",
                    help="also run the fused local path over a ragged plan (0 = automatic range)")
    args = ap.parse_args()
    res = []
    if args.pdl_pair:
        for c in args.case or ["C3_gqa4_B1_8192"]:
            for graph in (False, True):
                r = pdl_pair(c, graph=graph)
                print(json.dumps(r), flush=True)
                res.append(r)
        if args.json:
            with open(args.json, "w") as f:
                json.dump(res, f, indent=1)
        return
    for c in args.case or ["C3_gqa4_B1_8192", "C3_gqa4_B8_8192", "C2_mha_B64_2048"]:
        for rb in [None] + (args.ragged_bps or []):
            r = run(c, ragged_bps=rb)
            print(json.dumps(r), flush=True)
            res.append(r)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
