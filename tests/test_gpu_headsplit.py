"""NEXT row F2 on the GPU: head-granular attention-level migration (the paper's literal
"KV Cache split along the attention head dimension", Fig. 4) -- the
K/V pages of the offloaded kv-heads move into a compact cold pool (bit-exact vs the
oracle), each instance runs attention over its own head range into disjoint rows of one
output, and the concat equals full attention (oracle, north_star tolerances)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bs():
    import paper_2510_13223_b200 as m
    m.lib()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("d,hkv,G,c", [(128, 8, 4, 6), (64, 4, 2, 1), (128, 8, 1, 4)])
def test_head_split_migration_and_attention(bs, d, hkv, G, c):
    shape = synth.Shape(2, hkv * G, hkv, d)
    lens = (1, 100, 333, 2000)
    dense = synth.gen_dense(shape, lens, seed=d + G)
    ks = np.stack([np.zeros(len(lens)), np.asarray(lens)], 1).astype(np.int32)
    home_np = synth.place_shards(dense, ks, seed=3, spare_blocks=2)[0]
    nb = home_np.pool.shape[1]
    home = bs.KVPool(2, nb, hkv, d)
    home.data.copy_(_dev(home_np.pool))
    nh = hkv - c
    cold = bs.KVPool(2, nb, nh, d)
    cold_np = np.full((2, nb, 2, nh, 16, d), synth.DST_SENTINEL, dtype=np.uint16)
    cold.data.copy_(_dev(cold_np))
    ids = np.array(sorted({int(x) for x in home_np.block_tables.ravel() if x >= 0}), dtype=np.int32)
    idt = torch.from_numpy(ids).cuda()
    for layer in range(2):
        bs.kv_migrate_heads_layer(home, cold, layer, idt, idt, c, 0, nh)
        oracle.migrate_heads_layer(home_np.pool, cold_np, layer, ids, ids, c, 0, nh)
    torch.cuda.synchronize()
    assert np.array_equal(cold.data.cpu().view(torch.int16).numpy().view(np.uint16), cold_np)

    sc = synth.default_scale(d)
    B, hq = len(lens), hkv * G
    bt = torch.from_numpy(home_np.block_tables).cuda()
    ksd = torch.from_numpy(ks).cuda()
    for layer in range(2):
        q = _dev(dense.q[layer])
        o = torch.full((B, hq, d), float("nan"), device="cuda")
        m = torch.full((B, hq), float("nan"), device="cuda")
        l = torch.full((B, hq), float("nan"), device="cuda")
        for pool, plo, mlo, n in ((home, 0, 0, c), (cold, 0, c, nh)):
            wsn = bs.split_decode_attention_heads_workspace_size(pool, B, n, hkv, hq, bt.shape[1])
            ws = torch.zeros(max(16, wsn), dtype=torch.uint8, device="cuda")
            bs.split_decode_attention_heads(pool, layer, plo, mlo, n, hkv, q, bt, ksd, 0, sc, o, m, l, ws)
        out = torch.empty(B, hq, d, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(B, hq, device="cuda")
        bs.merge_partials([o], [m], [l], out, lse)          # n = 1: a pure bf16 conversion
        torch.cuda.synchronize()
        ref_o, ref_lse = oracle.attention_full([home_np.pool], [home_np.block_tables], layer,
                                               dense.q[layer], ks, sc)
        got = out.float().cpu().double().numpy()
        assert np.abs(got - ref_o).max() <= 2e-2
        rel = np.abs(got - ref_o).max(-1) / np.abs(ref_o).max(-1)
        assert rel.max() <= 1e-2
        assert np.abs(lse.cpu().double().numpy() - ref_lse).max() <= 1e-4
