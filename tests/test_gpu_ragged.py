"""Ragged plan path (bs_attention_ragged_plan + bs_split_decode_attention_local_ragged)
against the fp64 oracle: mixed lengths incl. empty requests / shards, unaligned splits,
G 1-8, d 64/128, 1-3 local shards, forced short ranges (many ranges per request) and the
automatic range; full-size C4 shape (Llama-2-70B GQA-8, 256 mixed-length requests, one
of 8 shards) on sampled requests; bitwise-deterministic reruns."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ABS_TOL, ROW_REL_TOL, LSE_TOL = 2e-2, 1e-2, 1e-4


@pytest.fixture(scope="module")
def bs():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2510_13223_b200 as m
    m.lib()
    return m


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def dev_i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def compare(out, lse, ref_o, ref_lse):
    got = out.float().cpu().double().numpy()
    gl = lse.cpu().double().numpy()
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isneginf(gl), ~fin) and np.all(got[~fin] == 0)
    err = np.abs(got - ref_o)
    assert err.max() <= ABS_TOL
    assert (err.max(-1)[fin] / np.abs(ref_o).max(-1)[fin]).max() <= ROW_REL_TOL
    assert np.abs(gl[fin] - ref_lse[fin]).max() <= LSE_TOL


@pytest.mark.parametrize("d,G", [(128, 1), (128, 4), (128, 8), (64, 2)])
@pytest.mark.parametrize("n_local", [1, 2, 3])
@pytest.mark.parametrize("bps", [16, 0])
def test_ragged_local_vs_oracle(bs, d, G, n_local, bps):
    shape = synth.Shape(1, 2 * G, 2, d)
    lens = (0, 1, 17, 100, 700, 2000, 3000, 5, 0, 640)
    dense = synth.gen_dense(shape, lens, seed=d + G + n_local)
    ks = synth.random_split(lens, n_local, seed=n_local + 5)
    shards = synth.place_shards(dense, ks, seed=G)
    pools = []
    for sh in shards:
        p = bs.KVPool(1, sh.pool.shape[1], shape.hkv, shape.d)
        p.data.copy_(dev_bf16(sh.pool))
        pools.append(p)
    bts = [dev_i32(sh.block_tables) for sh in shards]
    sc = synth.default_scale(d)
    B, hq = len(lens), shape.hq
    plan = bs.attention_ragged_plan(ks, list(range(n_local)), hq, shape.hkv, d,
                                    max_blocks_per_range=bps).to("cuda")
    ws = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device="cuda")
    q = dev_bf16(dense.q[0])
    ksd = dev_i32(ks)
    out = torch.full((B, hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((B, hq), float("nan"), device="cuda")
    bs.split_decode_attention_local_ragged(pools, 0, q, bts, list(range(n_local)), ksd, sc, plan,
                                           out, lse, ws)
    torch.cuda.synchronize()
    ref_o, ref_lse = oracle.attention_full([s.pool for s in shards], [s.block_tables for s in shards],
                                           0, dense.q[0], ks, sc)
    compare(out, lse, ref_o, ref_lse)
    out2 = torch.empty_like(out)
    bs.split_decode_attention_local_ragged(pools, 0, q, bts, list(range(n_local)), ksd, sc, plan,
                                           out2, None, ws)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), out2.view(torch.int16))


def test_full_size_c4_ragged_sampled(bs):
    """C4 at full size for one GPU's shard: Llama-2-70B GQA-8 (64/8 heads, d 128), 256
    mixed-length requests (Alpaca + LongBench-like), 8-way split -> shard 3 here."""
    shape = synth.Shape(1, 64, 8, 128)
    lens = synth.mixed_lengths(256, seed=0)
    ks8 = synth.block_aligned_split(lens, 8)
    ks = np.stack([np.zeros(256, np.int32), (ks8[:, 4] - ks8[:, 3]).astype(np.int32)], 1)
    case = synth.device_shards(shape, ks[:, 1], ks, seed=13, device="cuda", layers=1)
    pool = bs.KVPool(1, case.pools[0].shape[1], shape.hkv, shape.d, base=case.pools[0].reshape(-1))
    bts = [dev_i32(case.block_tables[0])]
    sc = synth.default_scale(shape.d)
    plan = bs.attention_ragged_plan(ks, [0], shape.hq, shape.hkv, shape.d).to("cuda")
    ws = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device="cuda")
    out = torch.empty(256, shape.hq, shape.d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(256, shape.hq, device="cuda")
    bs.split_decode_attention_local_ragged([pool], 0, case.q[0], bts, [0], dev_i32(ks), sc, plan,
                                           out, lse, ws)
    torch.cuda.synchronize()
    longest = int(np.argmax(ks[:, 1]))
    sample = sorted({longest, int(np.argmin(ks[:, 1])), 7, 100})
    sp, sbt, sks, sq = synth.extract_requests(case, sample, 0)
    ref_o, ref_lse = oracle.attention_full(sp, sbt, 0, sq, sks, sc)
    compare(out[sample], lse[sample], ref_o, ref_lse)


@pytest.mark.parametrize("d,G", [(128, 1), (128, 4), (128, 8), (64, 2)])
def test_packed_short_requests_vs_oracle(bs, d, G):
    """pack_short: requests of <= 8 blocks (here 0, 1, 5, 17, 100, 127, 128 tokens) run one warp
    per request, four to a CTA, beside ordinary items for the long ones; every output matches
    the oracle and reruns are bitwise identical.  Also with the PDL flag (graph, 3 layers)."""
    shape = synth.Shape(3, 2 * G, 2, d)
    lens = (0, 1, 5, 17, 100, 127, 128, 129, 700, 3000, 9, 64, 0, 33)
    dense = synth.gen_dense(shape, lens, seed=d + G)
    ks = np.stack([np.zeros(len(lens)), np.asarray(lens)], 1).astype(np.int32)
    shards = synth.place_shards(dense, ks, seed=G)
    pool = bs.KVPool(3, shards[0].pool.shape[1], shape.hkv, shape.d)
    pool.data.copy_(dev_bf16(shards[0].pool))
    bts = [dev_i32(shards[0].block_tables)]
    sc = synth.default_scale(d)
    B, hq = len(lens), shape.hq
    plan = bs.attention_ragged_plan(ks, [0], hq, shape.hkv, d, pack_short=True)
    n_packed = int(((plan.work[:, 3] & 0xFF) == 0).sum())
    assert n_packed == 3   # 11 requests of <= 8 blocks -> 3 packed items
    plan.to("cuda")
    ws = torch.zeros(max(16, plan.workspace_bytes), dtype=torch.uint8, device="cuda")
    ksd = dev_i32(ks)
    q = dev_bf16(dense.q)
    out = torch.full((3, B, hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((3, B, hq), float("nan"), device="cuda")

    def step():
        for layer in range(3):
            bs.split_decode_attention_local_ragged([pool], layer, q[layer], bts, [0], ksd, sc, plan,
                                                   out[layer], lse[layer], ws,
                                                   flags=bs.ATTN_PDL if layer else 0)
    step()
    torch.cuda.synchronize()
    first = (out.clone(), lse.clone())
    for layer in range(3):
        ref_o, ref_lse = oracle.attention_full([shards[0].pool], [shards[0].block_tables], layer,
                                               dense.q[layer], ks, sc)
        compare(out[layer], lse[layer], ref_o, ref_lse)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    out.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), first[0].view(torch.int16))
    assert torch.equal(lse, first[1])
