"""GPU parity of H7 (bs_kv_append_token, reading R-A9: the decoded token's K/V enters its
shard's paged cache before attention): bit-exact against the oracle's append on whole
pools, and the decode-step order append -> fused split attention + LSE merge against the
oracle's attention over the completed cache (tolerances of BASELINE.json's north star)."""
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


def host_u16(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def last_token_case(shape, lens, seed, layer, n_shards=1):
    """Cache laid out from the full dense KV with each request's last token (in the last
    shard) poisoned in ``layer``; returns what the append must restore."""
    dense = synth.gen_dense(shape, lens, seed)
    ks = (synth.block_aligned_split(lens, n_shards) if n_shards > 1 else
          np.stack([np.zeros(len(lens)), np.asarray(lens)], 1).astype(np.int32))
    shards = synth.place_shards(dense, ks, seed=seed)
    tail = shards[-1]
    pos = (ks[:, -1] - ks[:, -2] - 1).astype(np.int32)          # local index in the last shard
    partial = tail.pool.copy()
    for b, p in enumerate(pos):
        if p >= 0:
            partial[layer, tail.block_tables[b, p // 16], :, :, p % 16, :] = synth.BF16_NAN
    gl = np.asarray(lens) - 1
    k_new = np.stack([dense.k[b][layer, max(g, 0)] for b, g in enumerate(gl)])
    v_new = np.stack([dense.v[b][layer, max(g, 0)] for b, g in enumerate(gl)])
    return dense, ks, shards, partial, pos, k_new, v_new


@pytest.mark.parametrize("shape,lens", [
    (synth.Shape(2, 4, 2, 64), (37, 64, 129, 200, 17, 1)),
    (synth.Shape(2, 32, 32, 128), tuple(int(x) for x in
                                        np.random.default_rng(5).integers(1, 700, 64))),
    (synth.Shape(1, 64, 8, 128), (16, 32, 33, 4095, 4096, 4097)),
])
def test_append_bit_exact_vs_oracle(bs, shape, lens):
    layer = shape.n_layers - 1
    dense, ks, shards, partial, pos, k_new, v_new = last_token_case(shape, lens, 3, layer)
    pos[1] = -1                                        # skipped request keeps its poison
    ref = partial.copy()
    oracle.append_token(ref, layer, k_new, v_new, shards[0].block_tables, pos)
    L, nb = partial.shape[:2]
    pool = bs.KVPool(L, nb, shape.hkv, shape.d)
    pool.data.copy_(dev_bf16(partial))
    bs.kv_append_token(pool, layer, dev_bf16(k_new), dev_bf16(v_new),
                       dev_i32(shards[0].block_tables), dev_i32(pos))
    torch.cuda.synchronize()
    assert np.array_equal(host_u16(pool.data), ref)
    # every request but the skipped one now matches the cache laid out from the full KV
    full = shards[0].pool
    b, p = 1, int(ks[1, 1] - 1)
    blk = shards[0].block_tables[b, p // 16]
    got = host_u16(pool.data)
    got[layer, blk, :, :, p % 16, :] = full[layer, blk, :, :, p % 16, :]
    assert np.array_equal(got, full)


@pytest.mark.parametrize("n_shards", [1, 2])
def test_decode_step_append_then_attention(bs, n_shards):
    """One decode step of layer l in the product order: H7 append into the shard holding
    the sequence's end, then H4 + H6 fused over the co-located shards; equals the oracle's
    attention over the completed cache, which equals dense attention incl. the token."""
    shape = synth.Shape(1, 32, 8, 128)
    lens = (1, 16, 17, 500, 1024, 2049, 3000, 64)
    layer = 0
    dense, ks, shards, partial, pos, k_new, v_new = last_token_case(shape, lens, 11, layer, n_shards)
    pools = []
    for j, s in enumerate(shards):
        p = bs.KVPool(1, s.pool.shape[1], shape.hkv, shape.d)
        p.data.copy_(dev_bf16(partial if j == n_shards - 1 else s.pool))
        pools.append(p)
    bts = [dev_i32(s.block_tables) for s in shards]
    bs.kv_append_token(pools[-1], layer, dev_bf16(k_new), dev_bf16(v_new), bts[-1], dev_i32(pos))
    B, hq, d = len(lens), shape.hq, shape.d
    sc = synth.default_scale(d)
    ws_n = bs.split_decode_attention_local_workspace_size(pools, [t.shape[1] for t in bts], B, hq)
    ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device="cuda")
    out = torch.empty(B, hq, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, hq, device="cuda")
    bs.split_decode_attention_local(pools, layer, dev_bf16(dense.q[layer]), bts, list(range(n_shards)),
                                    dev_i32(ks), sc, out, lse, ws)
    torch.cuda.synchronize()
    ref_o, ref_lse = oracle.attention_full([s.pool for s in shards], [s.block_tables for s in shards],
                                           layer, dense.q[layer], ks, sc)
    got = out.float().cpu().double().numpy()
    err = np.abs(got - ref_o)
    assert err.max() <= ABS_TOL
    assert (err.max(-1) / np.abs(ref_o).max(-1)).max() <= ROW_REL_TOL
    assert np.abs(lse.cpu().double().numpy() - ref_lse).max() <= LSE_TOL


@pytest.mark.parametrize("shape,lens,n_pairs", [
    (synth.Shape(2, 4, 2, 64), (37, 64, 129, 200, 17, 1), 7),        # 2 KiB pages
    (synth.Shape(2, 32, 32, 128), (2048,) * 6 + (700, 5), 40),        # C2-like, 4 KiB pages
])
def test_migrate_append_one_launch_bit_exact(bs, shape, lens, n_pairs):
    """bs_kv_migrate_append_layer (H2 + H7 in one launch, the N=1 migration stream) equals
    the oracle's migrate of n chunk pairs into a sentinel-filled pool followed by its append
    into the source pool, byte for byte (both pools, every layer)."""
    layer = shape.n_layers - 1
    dense, ks, shards, partial, pos, k_new, v_new = last_token_case(shape, lens, 9, layer)
    pos[2] = -1
    L, nb = partial.shape[:2]
    spare = 2 * n_pairs
    src_np = np.concatenate([partial, synth.bf16_bits(torch.randn(
        (L, spare) + partial.shape[2:], generator=torch.Generator().manual_seed(4)))], axis=1)
    dst_np = np.full((L, n_pairs + 13) + partial.shape[2:], synth.DST_SENTINEL, dtype=np.uint16)
    rng = np.random.default_rng(2)
    s_ids = (nb + rng.permutation(spare)[:n_pairs]).astype(np.int32)   # outside the appends
    d_ids = rng.permutation(n_pairs + 13)[:n_pairs].astype(np.int32)
    ref_src, ref_dst = src_np.copy(), dst_np.copy()
    oracle.migrate_layer(ref_src, ref_dst, layer, s_ids, d_ids)
    oracle.append_token(ref_src, layer, k_new, v_new, shards[0].block_tables, pos)
    src = bs.KVPool(L, src_np.shape[1], shape.hkv, shape.d)
    src.data.copy_(dev_bf16(src_np))
    dst = bs.KVPool(L, dst_np.shape[1], shape.hkv, shape.d)
    dst.data.copy_(dev_bf16(dst_np))
    bs.kv_migrate_append_layer(src, dst, layer, dev_i32(s_ids), dev_i32(d_ids), src, dev_bf16(k_new),
                               dev_bf16(v_new), dev_i32(shards[0].block_tables), dev_i32(pos))
    torch.cuda.synchronize()
    assert np.array_equal(host_u16(dst.data), ref_dst)
    assert np.array_equal(host_u16(src.data), ref_src)
