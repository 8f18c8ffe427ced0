"""Pins for the fp64 oracle (DESIGN.md §Oracle pins).

Each test ties the oracle to something other than itself: numbers PAPER.md prints,
library routines (torch SDPA in fp64, scipy logsumexp), closed forms, invariants and
brute force on tiny inputs.  CPU only (-m "not gpu").
"""
import itertools
import math
import os

import numpy as np
import pytest
import torch
from scipy.special import logsumexp

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_eq15_17.txt")


def f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float64 (definition of bf16: the top half of an fp32)."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def sdpa_reference(dense, layer, scale):
    """Unsplit attention per request from torch's fp64 SDPA (a library routine) over the
    DENSE (pre-paging) K/V, plus lse from scipy.logsumexp over torch.matmul scores."""
    sh = dense.shape
    B = len(dense.seq_lens)
    o = np.zeros((B, sh.hq, sh.d))
    lse = np.zeros((B, sh.hq))
    for b in range(B):
        n = int(dense.seq_lens[b])
        q = torch.from_numpy(f64(dense.q[layer, b]))[None, :, None, :]           # [1,Hq,1,d]
        k = torch.from_numpy(f64(dense.k[b][layer])).permute(1, 0, 2)[None]     # [1,Hkv,n,d]
        v = torch.from_numpy(f64(dense.v[b][layer])).permute(1, 0, 2)[None]
        if n == 0:
            o[b] = 0.0
            lse[b] = -np.inf
            continue
        out = torch.nn.functional.scaled_dot_product_attention(
            q, k, v, scale=scale, enable_gqa=True)
        o[b] = out[0, :, 0, :].numpy()
        kk = k.repeat_interleave(sh.group, dim=1)                                 # [1,Hq,n,d]
        s = torch.matmul(q, kk.transpose(-1, -2))[0, :, 0, :].numpy() * scale     # [Hq,n]
        lse[b] = logsumexp(s, axis=-1)
    return o, lse


def unsplit_case(shape, lens, seed, n_needles=4):
    dense = synth.gen_dense(shape, lens, seed, n_needles=n_needles)
    ks = np.stack([np.zeros(len(lens)), np.asarray(lens)], axis=1).astype(np.int32)
    return dense, ks, synth.place_shards(dense, ks, seed=seed)


# ---------------------------------------------------------------------------- P1/P2

def test_golden_eq15_17_printed_values():
    rows = [ln.split() for ln in open(GOLDEN) if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 5
    for row in rows:
        name, args, printed, prec = row[0], row[1:-3], float(row[-2]), row[-1]
        if name == "d_head":
            got = int(args[0]) // int(args[1])
        elif name == "kv_bytes_per_token_layer":
            got = oracle.kv_bytes_per_token_layer(*map(int, args))
        elif name == "kv_bytes_per_token":
            got = oracle.kv_bytes_per_token(*map(int, args))
        elif name == "t_f_layer_ms":
            got = oracle.t_f_layer_ms(float(args[0]), float(args[1]), int(args[2]))
        elif name == "t_kv_ms":
            got = oracle.t_kv_ms(*map(float, args))
        else:
            raise AssertionError(name)
        if prec == "exact":
            assert got == printed, (name, got, printed)
        else:
            assert round(got, int(prec)) == printed, (name, got, printed)
    # the exact values behind the printed roundings (reading R-A17)
    assert oracle.t_f_layer_ms(270, 0.5, 32) == pytest.approx(4.21875, abs=1e-12)
    assert oracle.t_kv_ms(4096, 1000, 0.5, 200) == pytest.approx(0.08192, abs=1e-12)


GOLDEN_EQ34 = os.path.join(os.path.dirname(__file__), "golden", "paper_eq3_4_hand.txt")


def test_eq3_eq4_hand_worked_values():
    """eq. 3 (S_total = S_w + S_kv) and eq. 4 (T_layer ~= S_total / B_net + T_sync),
    PAPER.md:187-195: the oracle's helpers reproduce values worked by hand from model
    shapes (tests/golden/paper_eq3_4_hand.txt), and eq. 4's closed forms hold."""
    rows = [ln.split() for ln in open(GOLDEN_EQ34) if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 3
    for name, s_w, s_kv, s_tot, b_net, t_sync, t_layer in rows:
        s_w, s_kv, s_tot = int(s_w), int(s_kv), int(s_tot)
        assert oracle.layer_payload_bytes(s_w, s_kv) == s_tot, name
        assert oracle.t_layer_s(s_tot, float(b_net), float(t_sync)) == pytest.approx(
            float(t_layer), rel=1e-12), name
    # the hand sizes themselves, from the shapes (bf16): Llama-2-7B layer, 2048 tokens
    assert 2 * (4 * 4096 * 4096 + 3 * 4096 * 11008) == 404750336
    assert 2048 * oracle.kv_bytes_per_token_layer(32, 128) == 33554432
    # eq. 15's per-token size (printed) gives the Llama-3.1-8B S_kv
    assert 1000 * oracle.kv_bytes_per_token_layer(8, 128) == 4096000
    # eq. 4 closed forms: no payload -> T_sync; affine in S; inversely proportional to B
    assert oracle.t_layer_s(0.0, 1e9, 3e-3) == 3e-3
    t1 = oracle.t_layer_s(1e9, 1e11, 2e-3) - 2e-3
    t2 = oracle.t_layer_s(2e9, 1e11, 2e-3) - 2e-3
    assert t2 == pytest.approx(2 * t1, rel=1e-15) and t1 == pytest.approx(1e-2, rel=1e-15)
    assert oracle.t_layer_s(1e9, 2e11, 0.0) == pytest.approx(t1 / 2, rel=1e-15)


def test_pool_geometry_matches_eq15():
    # one (layer, block) chunk of the Llama-3.1-8B shape = 16 tokens x eq. 15's 4096 B
    assert oracle.chunk_elems(8, 16, 128) * 2 == 16 * oracle.kv_bytes_per_token_layer(8, 128)
    assert oracle.pool_bytes(32, 10, 8, 16, 128) == 32 * 10 * 16 * 4096


# ---------------------------------------------------------------------------- P3

@pytest.mark.parametrize("shape,lens", [
    (synth.TOY, synth.TOY_SEQ_LENS),
    (synth.Shape(2, 8, 2, 128), (1, 15, 16, 17, 300)),
    (synth.Shape(1, 4, 4, 64), (33, 5)),   # MHA, G = 1
    (synth.Shape(1, 8, 1, 64), (50,)),     # MQA, G = Hq
])
def test_attention_equals_torch_sdpa_fp64(shape, lens):
    dense, ks, shards = unsplit_case(shape, lens, seed=3)
    sc = synth.default_scale(shape.d)
    for layer in range(shape.n_layers):
        o, m, l = oracle.attention_shard(shards[0].pool, layer, dense.q[layer],
                                         shards[0].block_tables, ks, 0, sc)
        ref_o, ref_lse = sdpa_reference(dense, layer, sc)
        assert np.abs(o - ref_o).max() < 1e-12
        assert np.abs(m + np.log(l) - ref_lse).max() < 1e-12


def test_gqa_mapping_is_contiguous_groups():
    """A transposed head mapping (h % Hkv) would fail against repeat_interleave."""
    shape = synth.Shape(1, 4, 2, 64)
    dense, ks, shards = unsplit_case(shape, (40,), seed=5)
    sc = synth.default_scale(64)
    o, _, _ = oracle.attention_shard(shards[0].pool, 0, dense.q[0], shards[0].block_tables, ks, 0, sc)
    ref, _ = sdpa_reference(dense, 0, sc)
    assert np.abs(o - ref).max() < 1e-12
    wrong = dense.q[0][:, [0, 2, 1, 3]]  # heads 1 and 2 swapped => different kv head
    o2, _, _ = oracle.attention_shard(shards[0].pool, 0, wrong, shards[0].block_tables, ks, 0, sc)
    assert np.abs(o2[:, [0, 2, 1, 3]] - ref).max() > 1e-3


# ---------------------------------------------------------------------------- P4

def test_closed_form_zero_query():
    shape = synth.Shape(1, 4, 2, 64)
    lens = (1, 16, 37, 200)
    dense, ks, shards = unsplit_case(shape, lens, seed=11)
    q0 = np.zeros_like(dense.q[0])
    o, m, l = oracle.attention_shard(shards[0].pool, 0, q0, shards[0].block_tables, ks, 0, 0.125)
    for b, n in enumerate(lens):
        assert np.all(m[b] == 0.0)
        assert np.all(l[b] == float(n))                          # lse = ln n exactly
        vmean = f64(dense.v[b][0]).mean(axis=0)                  # [Hkv,d]
        for h in range(4):
            assert np.abs(o[b, h] - vmean[h // 2]).max() < 1e-12


def test_closed_form_single_token():
    shape = synth.Shape(1, 2, 1, 128)
    dense, ks, shards = unsplit_case(shape, (1,), seed=2, n_needles=0)
    sc = synth.default_scale(128)
    o, m, l = oracle.attention_shard(shards[0].pool, 0, dense.q[0], shards[0].block_tables, ks, 0, sc)
    v0 = f64(dense.v[0][0, 0, 0])
    k0 = f64(dense.k[0][0, 0, 0])
    for h in range(2):
        assert np.array_equal(o[0, h], v0)
        assert l[0, h] == 1.0
        assert m[0, h] == pytest.approx(sc * float(np.dot(f64(dense.q[0, 0, h]), k0)), abs=1e-12)


def test_closed_form_identical_keys_and_needle():
    shape = synth.Shape(1, 1, 1, 64)
    dense = synth.gen_dense(shape, (64,), seed=4, n_needles=0)
    dense.k[0][0, :] = dense.k[0][0, 0]                          # identical keys
    ks = np.array([[0, 64]], dtype=np.int32)
    sh = synth.place_shards(dense, ks, seed=4)[0]
    o, m, l = oracle.attention_shard(sh.pool, 0, dense.q[0], sh.block_tables, ks, 0, 0.125)
    assert l[0, 0] == pytest.approx(64.0, abs=1e-12)
    assert np.abs(o[0, 0] - f64(dense.v[0][0]).mean(axis=0)[0]).max() < 1e-12
    # needle: one key whose score is >= 50 above every other
    q = np.zeros((1, 1, 64), dtype=np.uint16)
    q[0, 0, 0] = 0x3F80                                           # 1.0
    dense.k[0][0, :, 0, :] = 0
    dense.k[0][0, 23, 0, 0] = 0x4348                              # 200.0 -> score 200*0.25 = 50
    sh = synth.place_shards(dense, ks, seed=4)[0]
    o, m, l = oracle.attention_shard(sh.pool, 0, q, sh.block_tables, ks, 0, 0.25)
    vneedle = f64(dense.v[0][0, 23, 0])
    tol = 64 * math.exp(-50) * np.abs(f64(dense.v[0][0])).max()
    assert np.abs(o[0, 0] - vneedle).max() <= tol + 1e-15
    assert m[0, 0] == 50.0


# ---------------------------------------------------------------------------- P5

@pytest.mark.parametrize("n_shards", [1, 2, 3, 4, 8])
def test_split_invariance_random_splits(n_shards):
    shape = synth.Shape(1, 8, 2, 64)
    lens = (0, 1, 16, 17, 77, 250)
    dense = synth.gen_dense(shape, lens, seed=20 + n_shards)
    sc = synth.default_scale(64)
    ref_o, ref_lse = sdpa_reference(dense, 0, sc)
    for trial in range(3):
        ks = synth.random_split(lens, n_shards, seed=100 * n_shards + trial)
        shards = synth.place_shards(dense, ks, seed=trial)
        o, lse = oracle.attention_full([s.pool for s in shards], [s.block_tables for s in shards],
                                       0, dense.q[0], ks, sc)
        assert np.array_equal(np.isneginf(lse), np.isneginf(ref_lse))
        fin = np.isfinite(ref_lse)
        assert np.abs(o - ref_o).max() < 1e-12
        assert np.abs(lse[fin] - ref_lse[fin]).max() < 1e-12
    assert np.all(o[0] == 0.0) and np.all(np.isneginf(lse[0]))   # seq_len 0 (R-A7)


def test_chained_protocol_equals_merge_and_sdpa():
    shape = synth.Shape(1, 4, 2, 64)
    lens = (37, 64, 129, 200, 5)
    dense = synth.gen_dense(shape, lens, seed=9)
    ks = synth.random_split(lens, 2, seed=1)
    ks[4, 1] = 0                                                    # empty hot shard
    shards = synth.place_shards(dense, ks, seed=9)
    sc = synth.default_scale(64)
    o_c, lse_c = oracle.chained_two_shard(shards[0].pool, shards[0].block_tables, shards[1].pool,
                                          shards[1].block_tables, 0, dense.q[0], ks, sc)
    o_m, lse_m = oracle.attention_full([s.pool for s in shards], [s.block_tables for s in shards],
                                       0, dense.q[0], ks, sc)
    ref_o, ref_lse = sdpa_reference(dense, 0, sc)
    assert np.abs(o_c - o_m).max() < 1e-12 and np.abs(o_c - ref_o).max() < 1e-12
    assert np.abs(lse_c - ref_lse).max() < 1e-12


def test_merge_edge_cases():
    d = 8
    o1 = np.arange(d, dtype=np.float64)[None, None]
    z = np.zeros((1, 1, d))
    # all shards empty
    o, lse = oracle.merge_partials([z, z], [np.full((1, 1), -np.inf)] * 2, [np.zeros((1, 1))] * 2)
    assert np.all(o == 0) and np.isneginf(lse).all()
    # one empty shard gets weight 0
    o, lse = oracle.merge_partials([z, o1], [np.full((1, 1), -np.inf), np.full((1, 1), 3.0)],
                                   [np.zeros((1, 1)), np.full((1, 1), 2.0)])
    assert np.array_equal(o, o1) and lse[0, 0] == pytest.approx(3.0 + math.log(2.0), abs=1e-15)
    # lse equals scipy logsumexp of the per-shard lse values
    rng = np.random.default_rng(0)
    m = rng.normal(size=(5, 3, 2)) * 10
    l = rng.uniform(0.5, 100, size=(5, 3, 2))
    oo = rng.normal(size=(5, 3, 2, d))
    o, lse = oracle.merge_partials(list(oo), list(m), list(l))
    ref = logsumexp(m + np.log(l), axis=0)
    assert np.abs(lse - ref).max() < 1e-12
    w = np.exp(m + np.log(l) - ref[None])
    assert np.abs(o - (w[..., None] * oo).sum(0)).max() < 1e-12


# ---------------------------------------------------------------------------- P6

def test_migrate_byte_identity_and_sentinel():
    dense, ks, shards = synth.toy_case(seed=0)
    src = shards[1]                                       # the offloaded shard (Fig. 4 KV2)
    nb_dst = 40
    dst = np.full((1, nb_dst) + src.pool.shape[2:], synth.DST_SENTINEL, dtype=np.uint16)
    alloc = oracle.Allocator(nb_dst)
    assert alloc.alloc(5) is not None                     # pre-existing tenant blocks 0..4
    src_ids, dst_ids, new_bt = [], [], np.full_like(src.block_tables, -1)
    for b in range(len(synth.TOY_SEQ_LENS)):
        row = [x for x in src.block_tables[b] if x >= 0]
        got = alloc.alloc(len(row))
        new_bt[b, :len(row)] = got
        src_ids += row
        dst_ids += list(got)
    assert dst_ids == list(range(5, 5 + len(dst_ids)))    # lowest-free-first (R-A12)
    oracle.migrate_layer(src.pool, dst, 0, src_ids, dst_ids)
    # byte identity through the block tables
    for b in range(len(synth.TOY_SEQ_LENS)):
        for i, x in enumerate(src.block_tables[b]):
            if x < 0:
                break
            assert np.array_equal(dst[0, new_bt[b, i]], src.pool[0, x])
    untouched = sorted(set(range(nb_dst)) - set(dst_ids))
    assert np.all(dst[:, untouched] == synth.DST_SENTINEL)
    # eq. 5: attention through the destination equals attention through the source, bitwise
    sc = synth.default_scale(64)
    a = oracle.attention_shard(src.pool, 0, dense.q[0], src.block_tables, ks, 1, sc)
    b_ = oracle.attention_shard(dst, 0, dense.q[0], new_bt, ks, 1, sc)
    for x, y in zip(a, b_):
        assert np.array_equal(x, y)


def test_allocator_policy_brute_force():
    rng = np.random.default_rng(1)
    for trial in range(200):
        nb = int(rng.integers(1, 12))
        used = rng.integers(0, 2, size=nb).astype(np.uint8)
        a = oracle.Allocator(nb)
        a.used[:] = used
        n = int(rng.integers(0, nb + 2))
        free_ids = [i for i in range(nb) if not used[i]]
        got = a.alloc(n)
        if n > len(free_ids):
            assert got is None and np.array_equal(a.used, used)     # all-or-nothing
        else:
            assert list(got) == free_ids[:n]                          # the n lowest free ids
            exp = used.copy()
            exp[free_ids[:n]] = 1
            assert np.array_equal(a.used, exp)
    a = oracle.Allocator(4)
    ids = a.alloc(3)
    assert not a.free([ids[0], ids[0]])                               # duplicate => error
    assert not a.free([3])                                            # not allocated
    assert not a.free([7])                                            # out of range
    assert list(a.used) == [1, 1, 1, 0]                               # no state change
    assert a.free([1]) and list(a.alloc(2)) == [1, 3]


# ---------------------------------------------------------------------------- P7

def test_toy_brute_force_all_aligned_two_way_splits():
    dense = synth.gen_dense(synth.TOY, synth.TOY_SEQ_LENS, seed=0)
    sc = synth.default_scale(64)
    ref_o, ref_lse = sdpa_reference(dense, 0, sc)
    choices = [list(range(0, n + 1, 16)) + ([n] if n % 16 else []) for n in synth.TOY_SEQ_LENS]
    count = 0
    for cuts in itertools.product(*[c[::2] if len(c) > 8 else c for c in choices]):
        ks = np.array([[0, c, n] for c, n in zip(cuts, synth.TOY_SEQ_LENS)], dtype=np.int32)
        shards = synth.place_shards(dense, ks, seed=count)
        o, lse = oracle.attention_full([s.pool for s in shards], [s.block_tables for s in shards],
                                       0, dense.q[0], ks, sc)
        assert np.abs(o - ref_o).max() < 1e-12 and np.abs(lse - ref_lse).max() < 1e-12
        count += 1
        if count >= 120:
            break
    assert count >= 100


# ---------------------------------------------------------------------------- NEXT F2

def test_migrate_heads_pages_and_head_split_attention():
    """Head-granular migration: moved pages are byte-identical, other
    heads and blocks keep their sentinel, and attention for the migrated kv-heads read
    from the compact cold pool equals the same heads read from the full pool (eq. 5);
    concatenating the two head groups reproduces full attention (torch SDPA)."""
    shape = synth.Shape(1, 8, 4, 64)                      # G = 2
    lens = (37, 70)
    dense, ks, shards = unsplit_case(shape, lens, seed=12)
    home = shards[0]
    c0, nh = 3, 1                                         # migrate kv-head 3 only
    nb = home.pool.shape[1]
    cold = np.full((1, nb, 2, nh, 16, 64), synth.DST_SENTINEL, dtype=np.uint16)
    ids = np.array([x for x in home.block_tables.ravel() if x >= 0], dtype=np.int32)
    oracle.migrate_heads_layer(home.pool, cold, 0, ids, ids, c0, 0, nh)
    for x in range(nb):
        if x in set(ids.tolist()):
            assert np.array_equal(cold[0, x, :, 0], home.pool[0, x, :, c0])
        else:
            assert np.all(cold[0, x] == synth.DST_SENTINEL)
    sc = synth.default_scale(64)
    o_full, m_full, l_full = oracle.attention_shard(home.pool, 0, dense.q[0], home.block_tables, ks, 0, sc)
    G = 2
    q_cold = np.ascontiguousarray(dense.q[0][:, c0 * G:(c0 + nh) * G])
    o_c, m_c, l_c = oracle.attention_shard(cold, 0, q_cold, home.block_tables, ks, 0, sc)
    assert np.array_equal(o_c, o_full[:, c0 * G:(c0 + nh) * G])
    assert np.array_equal(m_c, m_full[:, c0 * G:(c0 + nh) * G])
    ref, _ = sdpa_reference(dense, 0, sc)
    cat = np.concatenate([o_full[:, :c0 * G], o_c], axis=1)   # merge = concat for a head split
    assert np.abs(cat - ref).max() < 1e-12


# ---------------------------------------------------------------------------- H7 append

def append_case(seed=0, lens=(37, 64, 129, 200, 17), layer=1):
    """A 2-layer toy-shaped cache laid out from the FULL dense KV, and the same cache with
    each request's last token (the one being decoded, reading R-A9) not yet written in
    ``layer`` (its slot poisoned with bf16 NaN).  Positions cover a mid-block slot (36),
    the last slot of a block (63), the first slot of a new block (128, 16) and 199."""
    shape = synth.Shape(n_layers=2, hq=4, hkv=2, d=64)
    dense = synth.gen_dense(shape, lens, seed)
    ks = np.stack([np.zeros(len(lens)), np.asarray(lens)], axis=1).astype(np.int32)
    full = synth.place_shards(dense, ks, seed=seed)[0]
    pos = np.asarray(lens, dtype=np.int32) - 1
    partial = full.pool.copy()
    for b, p in enumerate(pos):
        partial[layer, full.block_tables[b, p // 16], :, :, p % 16, :] = synth.BF16_NAN
    k_new = np.stack([dense.k[b][layer, p] for b, p in enumerate(pos)])   # [B][Hkv][d]
    v_new = np.stack([dense.v[b][layer, p] for b, p in enumerate(pos)])
    return dense, ks, full, partial, pos, k_new, v_new


def test_append_token_completes_the_paged_cache():
    """(H7) Appending each request's decoded token reproduces, byte for byte, the cache
    laid out from the full dense KV (pins block = bt[pos // 16], slot = pos % 16, K before
    V, head order, the layer); every other byte is untouched; attention over the completed
    cache equals torch's fp64 SDPA over the dense KV including that token."""
    layer = 1
    dense, ks, full, partial, pos, k_new, v_new = append_case(layer=layer)
    before = partial.copy()
    oracle.append_token(partial, layer, k_new, v_new, full.block_tables, pos)
    assert np.array_equal(partial, full.pool)
    assert np.array_equal(partial[0], before[0])          # other layer untouched
    sc = synth.default_scale(64)
    o, m, l = oracle.attention_shard(partial, layer, dense.q[layer], full.block_tables, ks, 0, sc)
    ref_o, ref_lse = sdpa_reference(dense, layer, sc)
    assert np.abs(o - ref_o).max() < 1e-12
    assert np.abs(m + np.log(l) - ref_lse).max() < 1e-12


def test_append_token_negative_position_skips():
    layer = 1
    dense, ks, full, partial, pos, k_new, v_new = append_case(layer=layer)
    skip = pos.copy()
    skip[2] = -1
    oracle.append_token(partial, layer, k_new, v_new, full.block_tables, skip)
    b, p = 2, int(pos[2])
    blk = full.block_tables[b, p // 16]
    assert np.all(partial[layer, blk, :, :, p % 16, :] == synth.BF16_NAN)
    partial[layer, blk, :, :, p % 16, :] = full.pool[layer, blk, :, :, p % 16, :]
    assert np.array_equal(partial, full.pool)
