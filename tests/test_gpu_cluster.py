"""Cluster merge of split-K ranges: single-wave launches whose (request,
kv-head) pairs are cut into 2..16 CTA ranges run each pair's ranges as one thread-block
cluster; the non-leader CTAs st.async their partial into the leader's shared memory and the
leader merges (eq. 10) from there instead of the workspace.

Checked here: the launch really takes the cluster path (bs_attention_last_launch), its
outputs equal the workspace merge (BS_ATTN_NO_CLUSTER) bit for bit -- same range cut, same
merge arithmetic and order (R-A14) -- and the fp64 oracle within the north-star tolerances,
for every G and d, ragged / unaligned / empty requests, one and two local shards, the
per-shard partial API, repeated launches and CUDA-graph replay."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ABS_TOL, ROW_REL_TOL, LSE_TOL, PART_TOL = 2e-2, 1e-2, 1e-4, 5e-3


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


def host_case(bs, shape, lens, n_shards, seed):
    dense = synth.gen_dense(shape, lens, seed=seed)
    ks = synth.random_split(lens, n_shards, seed=seed) if n_shards > 1 else \
        np.stack([np.zeros(len(lens)), np.asarray(lens)], 1).astype(np.int32)
    shards = synth.place_shards(dense, ks, seed=seed + 1)
    pools = []
    for s in shards:
        p = bs.KVPool(shape.n_layers, s.pool.shape[1], shape.hkv, shape.d)
        p.data.copy_(dev_bf16(s.pool))
        pools.append(p)
    return dense, ks, shards, pools


def local_run(bs, pools, bts, ks, q, scale, flags, layer=0):
    B, hq, d = q.shape
    ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
        pools, [t.shape[1] for t in bts], B, hq)), dtype=torch.uint8, device="cuda")
    out = torch.full((B, hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((B, hq), float("nan"), device="cuda")
    bs.split_decode_attention_local(pools, layer, q, bts, list(range(len(pools))), ks, scale, out,
                                    lse, ws, flags=flags)
    info = bs.attention_last_launch()
    torch.cuda.synchronize()
    return out, lse, info


def check_merged(shards, ks, q_u16, scale, out, lse, layer=0):
    parts = [oracle.attention_shard(s.pool, layer, q_u16, s.block_tables, ks, j, scale)
             for j, s in enumerate(shards)]
    ref_o, ref_lse = oracle.merge_partials(*zip(*parts))
    got = out.float().cpu().double().numpy()
    gl = lse.cpu().double().numpy()
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isneginf(gl), ~fin)
    assert np.all(got[~fin] == 0)
    err = np.abs(got - ref_o)
    assert err.max() <= ABS_TOL, err.max()
    if fin.any():
        rel = err.max(axis=-1)[fin] / np.maximum(np.abs(ref_o).max(axis=-1)[fin], 1e-30)
        assert rel.max() <= ROW_REL_TOL, rel.max()
        assert np.abs(gl[fin] - ref_lse[fin]).max() <= LSE_TOL


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_cluster_merge_equals_workspace_merge_and_oracle(bs, d, G):
    """48 (request, kv-head) pairs over two local shards: a one-wave plan has <= 9 ranges per
    pair; ragged / unaligned / tiny / empty requests (empty ranges send empty partials)."""
    shape = synth.Shape(1, 8 * G, 8, d)
    lens = (3000, 0, 1, 17, 999, 2048)
    dense, ks, shards, pools = host_case(bs, shape, lens, 2, seed=31 * G + d)
    bts = [dev_i32(s.block_tables) for s in shards]
    ksd = dev_i32(ks)
    q = dev_bf16(dense.q[0])
    sc = synth.default_scale(d)
    o_cl, l_cl, info = local_run(bs, pools, bts, ksd, q, sc, 0)
    o_ws, l_ws, info_ws = local_run(bs, pools, bts, ksd, q, sc, bs.ATTN_NO_CLUSTER)
    cl_max = int(os.environ.get("BS_ATTN_CLUSTER_MAX", "8"))
    assert 2 <= info["ranges"] <= 16 and info["tensor_cores"] == 1, info
    assert info["cluster"] == (1 if info["ranges"] <= cl_max else 0), info
    assert info_ws["cluster"] == 0 and info_ws["ranges"] == info["ranges"]
    assert torch.equal(o_cl.view(torch.int16), o_ws.view(torch.int16))
    assert torch.equal(l_cl, l_ws)
    check_merged(shards, ks, dense.q[0], sc, o_cl, l_cl)


@pytest.mark.parametrize("B", [1, 2, 8])
def test_c3_per_gpu_shard_cluster(bs, B):
    """The C3 per-GPU shard (Llama-3-8B GQA-4, 8192 tokens per request = a 4-way split of
    32k): B=8 cuts each (request, kv-head) into 4 ranges (4-CTA clusters); B=1 into 16 --
    above the default cluster cap (8), so the workspace merge; with BS_ATTN_CLUSTER_MAX=16
    (test below) 16-CTA non-portable clusters.  Repeated launches stay identical."""
    shape = synth.Shape(1, 32, 8, 128)
    lens = np.full(B, 8192)
    ks = np.stack([np.zeros(B), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=40 + B, device="cuda")
    pools = [bs.KVPool(1, p.shape[1], shape.hkv, shape.d, base=p.reshape(-1)) for p in case.pools]
    bts = [torch.from_numpy(b).cuda() for b in case.block_tables]
    ksd = torch.from_numpy(ks).cuda()
    sc = synth.default_scale(128)
    o1, l1, info = local_run(bs, pools, bts, ksd, case.q[0], sc, 0)
    o2, l2, _ = local_run(bs, pools, bts, ksd, case.q[0], sc, 0)
    o3, l3, _ = local_run(bs, pools, bts, ksd, case.q[0], sc, bs.ATTN_NO_CLUSTER)
    cl_max = int(os.environ.get("BS_ATTN_CLUSTER_MAX", "8"))
    assert info["stages"] == 2 and info["pdl"] == 0, info   # no PDL flag: 2-stage ring
    if B == 1:
        assert info["ranges"] == 16, info
    assert info["cluster"] == (1 if info["ranges"] <= cl_max else 0), info
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)) and torch.equal(l1, l2)
    assert torch.equal(o1.view(torch.int16), o3.view(torch.int16)) and torch.equal(l1, l3)
    req = [0, B - 1] if B > 1 else [0]
    sp, sbt, sks, sq = synth.extract_requests(case, req, 0)
    ref_o, ref_lse = oracle.attention_full(sp, sbt, 0, sq, sks, sc)
    got = o1[req].float().cpu().double().numpy()
    assert np.abs(got - ref_o).max() <= ABS_TOL
    assert np.abs(l1[req].cpu().double().numpy() - ref_lse).max() <= LSE_TOL


def test_partial_api_cluster_matches_oracle(bs):
    """bs_split_decode_attention (per-shard partial triple, not merged) on the cluster path:
    the leader writes (o~, m, l) of the whole shard."""
    shape = synth.Shape(1, 32, 8, 128)
    lens = (6000, 333, 1, 0, 4000, 17)
    dense, ks, shards, pools = host_case(bs, shape, lens, 1, seed=5)
    bt = dev_i32(shards[0].block_tables)
    B, hq, d = dense.q[0].shape
    o = torch.full((B, hq, d), float("nan"), device="cuda")
    m = torch.full((B, hq), float("nan"), device="cuda")
    l = torch.full((B, hq), float("nan"), device="cuda")
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pools[0], B, hq, bt.shape[1])),
                     dtype=torch.uint8, device="cuda")
    sc = synth.default_scale(d)
    bs.split_decode_attention(pools[0], 0, dev_bf16(dense.q[0]), bt, dev_i32(ks), 0, sc, o, m, l, ws)
    info = bs.attention_last_launch()
    torch.cuda.synchronize()
    assert info["cluster"] == 1 and info["ranges"] >= 2, info
    ro, rm, rl = oracle.attention_shard(shards[0].pool, 0, dense.q[0], shards[0].block_tables, ks, 0, sc)
    o, m, l = o.cpu().double().numpy(), m.cpu().double().numpy(), l.cpu().double().numpy()
    ne = rl > 0
    assert np.array_equal(l > 0, ne) and np.all(np.isneginf(m[~ne])) and np.all(o[~ne] == 0)
    assert np.abs(o - ro).max() <= PART_TOL
    assert np.abs((m + np.log(l))[ne] - (rm + np.log(rl))[ne]).max() <= LSE_TOL


def test_cluster_graph_replay_equals_eager(bs):
    """4 layers of C3 B=1 launches back to back, captured in a CUDA graph: replay == eager."""
    shape = synth.Shape(4, 32, 8, 128)
    lens = np.full(1, 8192)
    ks = np.stack([np.zeros(1), lens], 1).astype(np.int32)
    case = synth.device_shards(shape, lens, ks, seed=9, device="cuda")
    pools = [bs.KVPool(shape.n_layers, p.shape[1], shape.hkv, shape.d, base=p.reshape(-1))
             for p in case.pools]
    bts = [torch.from_numpy(b).cuda() for b in case.block_tables]
    ksd = torch.from_numpy(ks).cuda()
    sc = synth.default_scale(128)
    L = shape.n_layers
    ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(pools, [bts[0].shape[1]], 1, 32)),
                     dtype=torch.uint8, device="cuda")
    out = torch.zeros((L, 1, 32, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((L, 1, 32), device="cuda")

    def step():
        for layer in range(L):
            bs.split_decode_attention_local(pools, layer, case.q[layer], bts, [0], ksd, sc, out[layer],
                                            lse[layer], ws)
    step()
    torch.cuda.synchronize()
    o_e, l_e = out.clone(), lse.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    out.fill_(float("nan"))
    lse.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), o_e.view(torch.int16)) and torch.equal(lse, l_e)
    sp, sbt, sks, sq = synth.extract_requests(case, [0], L - 1)
    ref_o, ref_lse = oracle.attention_full(sp, sbt, 0, sq, sks, sc)
    assert np.abs(out[L - 1].float().cpu().double().numpy() - ref_o).max() <= ABS_TOL
    assert np.abs(lse[L - 1].cpu().double().numpy() - ref_lse).max() <= LSE_TOL


def test_sixteen_cta_clusters_subprocess():
    """BS_ATTN_CLUSTER_MAX=16 (read once per process): the C3 B=1 launch runs 16-CTA
    clusters, the small cases their 9-range clusters, and all still equal the workspace
    merge and the oracle."""
    env = dict(os.environ, BS_ATTN_CLUSTER_MAX="16")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "test_c3_per_gpu_shard_cluster and 1 or test_cluster_merge_equals"],
                       env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "9 passed" in r.stdout, r.stdout[-2000:]


_DUMP = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2510_13223_b200 as bs, synth
shape = synth.Shape(3, 32, 8, 128)
lens = np.array([8192, 5000])
ks = np.stack([np.zeros(2), lens], 1).astype(np.int32)
case = synth.device_shards(shape, lens, ks, seed=77, device="cuda")
pools = [bs.KVPool(3, p.shape[1], 8, 128, base=p.reshape(-1)) for p in case.pools]
bts = [torch.from_numpy(b).cuda() for b in case.block_tables]
ksd = torch.from_numpy(ks).cuda()
ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(pools, [bts[0].shape[1]], 2, 32)),
                 dtype=torch.uint8, device="cuda")
out = torch.empty(3, 2, 32, 128, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(3, 2, 32, device="cuda")
infos = []
for layer in range(3):
    bs.split_decode_attention_local(pools, layer, case.q[layer], bts, [0], ksd, synth.default_scale(128),
                                    out[layer], lse[layer], ws, flags=bs.ATTN_PDL if layer else 0)
    infos.append(bs.attention_last_launch())
torch.cuda.synchronize()
np.savez({path!r}, out=out.view(torch.int16).cpu().numpy(), lse=lse.cpu().numpy(),
         stages=np.array([i["stages"] for i in infos]), pdl=np.array([i["pdl"] for i in infos]))
"""


def test_deep_ring_variant_bitwise_equals_two_stage(tmp_path):
    """The one-CTA-per-SM 6-stage variant (PDL launches) changes only how far each warp's
    TMA ring runs ahead, not which blocks a warp folds in which order: its outputs equal the
    2-stage kernel's bit for bit (BS_ATTN_DEEP=0, separate processes: the switch is read
    once)."""
    import os.path
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for deep in ("1", "0"):
        path = str(tmp_path / f"deep{deep}.npz")
        env = dict(os.environ, BS_ATTN_DEEP=deep)
        r = subprocess.run([sys.executable, "-c", _DUMP.format(root=root, path=path)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[deep] = np.load(path)
    # layer 0 (no PDL flag) runs the 2-stage ring, the PDL layers the 6-stage one
    assert list(res["1"]["stages"]) == [2, 6, 6] and list(res["0"]["stages"]) == [2, 2, 2]
    assert list(res["1"]["pdl"]) == [0, 1, 1]
    assert np.array_equal(res["1"]["out"], res["0"]["out"])
    assert np.array_equal(res["1"]["lse"], res["0"]["lse"])



@pytest.mark.parametrize("seed", range(12))
def test_merge_paths_fuzz(bs, seed):
    """Random shapes through the fused local launch, two consecutive layers with the decode-
    step flag on the second: whatever merge / launch features the launch picks (cluster or
    last arriver, PDL trigger mode, 6-stage ring), the outputs equal the plain launch with
    the workspace merge (BS_ATTN_NO_CLUSTER, no PDL) bitwise and the oracle within the
    tolerances."""
    rng = np.random.default_rng(500 + seed)
    G = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    hkv = int(rng.choice([1, 2, 4, 8]))
    shape = synth.Shape(2, hkv * G, hkv, d)
    B = int(rng.integers(1, 9))
    lens = [int(x) for x in rng.choice([0, 1, 16, 17, 300, 1000, 4000, 9000], size=B)]
    n = int(rng.integers(1, 4))
    dense, ks, shards, pools = host_case(bs, shape, lens, n, seed=seed)
    bts = [dev_i32(s.block_tables) for s in shards]
    ksd = dev_i32(ks)
    sc = synth.default_scale(d)
    outs = {}
    for mode, flags in (("plain", bs.ATTN_NO_CLUSTER), ("features", bs.ATTN_PDL)):
        o = torch.full((2, B, shape.hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
        l = torch.full((2, B, shape.hq), float("nan"), device="cuda")
        ws = torch.zeros(max(16, bs.split_decode_attention_local_workspace_size(
            pools, [t.shape[1] for t in bts], B, shape.hq)), dtype=torch.uint8, device="cuda")
        for layer in range(2):
            bs.split_decode_attention_local(pools, layer, dev_bf16(dense.q[layer]), bts, list(range(len(pools))),
                                            ksd, sc, o[layer], l[layer], ws,
                                            flags=flags if (layer or mode == "plain") else 0)
        torch.cuda.synchronize()
        outs[mode] = (o, l)
    assert torch.equal(outs["plain"][0].view(torch.int16), outs["features"][0].view(torch.int16))
    assert torch.equal(outs["plain"][1], outs["features"][1])
    for layer in range(2):
        check_merged(shards, ks, dense.q[layer], sc, outs["features"][0][layer], outs["features"][1][layer],
                     layer=layer)
