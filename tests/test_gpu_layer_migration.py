"""NEXT row F3 on the GPU: layer-level migration (Fig. 3, eqs. 3-5) --
the KV of a contiguous layer range in one launch plus the layers' weight tensors,
bit-exact against the oracle, and eq. 5's invariance: attention of every migrated layer
read on the destination equals the source, bitwise."""
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


def test_layer_range_migration_with_weights(bs):
    shape = synth.Shape(6, 8, 2, 128)
    lens = (40, 513, 1000)
    dense = synth.gen_dense(shape, lens, seed=8)
    ks = np.stack([np.zeros(3), np.asarray(lens)], 1).astype(np.int32)
    src_np = synth.place_shards(dense, ks, seed=8, spare_blocks=5)[0]
    nb = src_np.pool.shape[1]
    src = bs.KVPool(6, nb, 2, 128)
    src.data.copy_(_dev(src_np.pool))
    nbd = nb + 9
    dst_np = np.full((6, nbd, 2, 2, 16, 128), synth.DST_SENTINEL, dtype=np.uint16)
    dst = bs.KVPool(6, nbd, 2, 128)
    dst.data.copy_(_dev(dst_np))
    ids = sorted({int(x) for x in src_np.block_tables.ravel() if x >= 0})
    new = {x: i + 7 for i, x in enumerate(ids)}            # a different placement
    s = np.array(ids, dtype=np.int32)
    t = np.array([new[x] for x in ids], dtype=np.int32)
    w_src = [torch.randn(4096, 512, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    w_dst = [torch.zeros_like(w) for w in w_src]
    payload = bs.migrate_layers(src, dst, 2, 3, torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda(),
                                weights=list(zip(w_src, w_dst)))
    torch.cuda.synchronize()
    oracle.migrate_layers(src_np.pool, dst_np, 2, 3, s, t)
    assert np.array_equal(dst.data.cpu().view(torch.int16).numpy().view(np.uint16), dst_np)
    assert all(torch.equal(a, b) for a, b in zip(w_src, w_dst))
    s_kv = 3 * len(ids) * src.chunk_bytes
    assert payload == oracle.layer_payload_bytes(sum(w.numel() * 2 for w in w_src), s_kv)
    # eq. 5: y_l = f_l(x_l; W_l, KV_l) unchanged after migration -- attention per layer
    bt_new = np.vectorize(lambda x: new.get(int(x), -1))(src_np.block_tables).astype(np.int32)
    sc = synth.default_scale(128)
    for layer in (2, 3, 4):
        q = _dev(dense.q[layer])
        outs = []
        for pool, bt in ((src, src_np.block_tables), (dst, bt_new)):
            o = torch.empty(3, 8, 128, device="cuda")
            m = torch.empty(3, 8, device="cuda")
            l = torch.empty(3, 8, device="cuda")
            ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(pool, 3, 8, bt.shape[1])),
                             dtype=torch.uint8, device="cuda")
            bs.split_decode_attention(pool, layer, q, torch.from_numpy(bt).cuda(),
                                      torch.from_numpy(ks).cuda(), 0, sc, o, m, l, ws)
            outs.append((o, m, l))
        torch.cuda.synchronize()
        for x, y in zip(*outs):
            assert torch.equal(x, y)
