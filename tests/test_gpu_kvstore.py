"""NEXT row F1 on the GPU: Global KV Cache Store CPU tier (pinned host pool) and the
three-stage layer-wise pipeline (Fig. 6).  Fetch (HtoD) and store
(DtoH) are bit-exact against the oracle's migrate; the pipeline's compute (split decode
attention over a resident batch) matches the oracle while fetch/store run beside it."""
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


def _rand(shape, L, nb, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 65536, (L, nb, 2, shape.hkv, 16, shape.d), generator=g,
                         dtype=torch.int32).to(torch.int16).numpy().view(np.uint16)


def _u16(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _fill(pool, arr):
    pool.data.copy_(torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16))


def test_host_pool_needs_pinned_memory(bs):
    with pytest.raises(ValueError):
        bs.KVPool(1, 4, 2, 64, host=True, base=torch.empty(4 * 2 * 2 * 16 * 64, dtype=torch.bfloat16))
    p = bs.KVPool(1, 4, 2, 64, host=True)
    assert p.data.is_pinned() and p.alloc(2) == [0, 1]
    with pytest.raises(bs.BSError):   # attention never reads the host tier
        o = torch.empty(1, 2, 64, device="cuda")
        m = torch.empty(1, 2, device="cuda")
        bs.split_decode_attention(p, 0, torch.zeros(1, 2, 64, dtype=torch.bfloat16, device="cuda"),
                                  torch.zeros(1, 1, dtype=torch.int32, device="cuda"),
                                  torch.tensor([[0, 5]], dtype=torch.int32, device="cuda"), 0, 0.1,
                                  o, m, m)


@pytest.mark.parametrize("engine", ["sm", "ce", "staged"])
@pytest.mark.parametrize("d,hkv", [(128, 8), (64, 2)])
def test_fetch_and_store_bit_exact(bs, d, hkv, engine):
    from paper_2510_13223_b200.kvstore import KVStore
    shape = synth.Shape(3, hkv, hkv, d)
    store = KVStore(3, 64, hkv, d)
    s_np = _rand(shape, 3, 64, 1)
    _fill(store.pool, s_np)
    dev = bs.KVPool(3, 80, hkv, d)
    d_np = np.full((3, 80, 2, hkv, 16, d), synth.DST_SENTINEL, dtype=np.uint16)
    _fill(dev, d_np)
    si = np.array([63, 0, 5, 6, 7, 17, 40], dtype=np.int32)     # 5,6,7 -> 2,3,4: a coalesced run
    di = np.array([1, 79, 2, 3, 4, 60, 50], dtype=np.int32)
    ids = (lambda a: torch.from_numpy(a).cuda()) if engine == "sm" else list
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        if engine == "staged":   # store runs [63] [0] [5..7] [17] [40] -> staging -> scatter
            fp = store.prepare(dev, list(si), list(di))
            assert [r[1] for r in fp.runs] == [1, 1, 3, 1, 1]
        for layer in range(3):
            if engine == "staged":
                store.fetch_staged(dev, layer, fp, stream=stream)
            else:
                store.fetch_layer(dev, layer, ids(si), ids(di), engine=engine)
    for layer in range(3):
        oracle.migrate_layer(s_np, d_np, layer, si, di)
    torch.cuda.synchronize()
    assert np.array_equal(_u16(dev.data), d_np)
    # store different device blocks back into free store blocks
    src = np.array([1, 79], dtype=np.int32)
    dst = np.array([10, 11], dtype=np.int32)
    if engine == "staged":
        store.store_staged(dev, 2, store.prepare(dev, list(dst), list(src)))
    else:
        store.store_layer(dev, 2, ids(src), ids(dst), engine=engine)
    torch.cuda.synchronize()
    oracle.migrate_layer(d_np, s_np, 2, src, dst)
    assert np.array_equal(_u16(store.pool.data), s_np)


@pytest.mark.parametrize("engine", ["sm", "ce", "staged"])
def test_three_stage_pipeline(bs, engine):
    from paper_2510_13223_b200.kvstore import KVStore, ThreeStagePipeline
    shape = synth.Shape(3, 8, 2, 128)
    lens = (300, 77, 1000)
    dense = synth.gen_dense(shape, lens, seed=4)
    ks = np.stack([np.zeros(3), np.asarray(lens)], 1).astype(np.int32)
    res = synth.place_shards(dense, ks, seed=4, spare_blocks=40)[0]
    nb = res.pool.shape[1]
    dev = bs.KVPool(3, nb, shape.hkv, shape.d)
    _fill(dev, res.pool)
    free = [i for i in range(nb) if not res.used[i]]
    store = KVStore(3, 100, shape.hkv, shape.d)
    s_np = _rand(shape, 3, 100, 9)
    _fill(store.pool, s_np)
    f_store = np.arange(20, dtype=np.int32)           # prefix blocks to fetch ...
    f_dev = np.array(free[:20], dtype=np.int32)        # ... into free device blocks
    used = [i for i in range(nb) if res.used[i]][:12]
    st_dev = np.array(used, dtype=np.int32)            # resident blocks stored back ...
    st_store = np.arange(60, 72, dtype=np.int32)       # ... into free store blocks
    q = torch.from_numpy(dense.q.view(np.int16)).view(torch.bfloat16).cuda()
    bt = torch.from_numpy(res.block_tables).cuda()
    ksd = torch.from_numpy(ks).cuda()
    sc = synth.default_scale(128)
    o = torch.empty(3, 3, 8, 128, device="cuda")
    m = torch.empty(3, 3, 8, device="cuda")
    l = torch.empty(3, 3, 8, device="cuda")
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(dev, 3, 8, bt.shape[1])),
                     dtype=torch.uint8, device="cuda")

    def compute(layer):
        bs.split_decode_attention(dev, layer, q[layer], bt, ksd, 0, sc, o[layer], m[layer], l[layer], ws)

    if engine == "sm":
        fp = (torch.from_numpy(f_store).cuda(), torch.from_numpy(f_dev).cuda())
        sp = (torch.from_numpy(st_dev).cuda(), torch.from_numpy(st_store).cuda())
    else:
        fp, sp = (list(f_store), list(f_dev)), (list(st_dev), list(st_store))
    pipe = ThreeStagePipeline(store, dev, 3, compute, fetch_pairs=fp, store_pairs=sp, engine=engine)
    pipe.enqueue()
    torch.cuda.synchronize()
    d_np = res.pool.copy()
    for layer in range(3):
        oracle.migrate_layer(s_np, d_np, layer, f_store, f_dev)
        oracle.migrate_layer(res.pool, s_np, layer, st_dev, st_store)
        ro, rm, rl = oracle.attention_shard(res.pool, layer, dense.q[layer], res.block_tables, ks, 0, sc)
        assert np.abs(o[layer].cpu().double().numpy() - ro).max() <= 1e-3
        assert np.abs((m[layer] + l[layer].log()).cpu().double().numpy() - (rm + np.log(rl))).max() <= 1e-4
    got_dev = _u16(dev.data)
    assert np.array_equal(got_dev[:, :, :, :, :, :], d_np)
    assert np.array_equal(_u16(store.pool.data), s_np)


def test_c5_prefix_hits_fetched_then_attended(bs):
    """C5-shaped (bursty, prefix hits from the Global KV Cache Store):
    each request's first half (r = 0.5) lives only in the host store; the three-stage
    pipeline fetches it layer by layer into the device blocks the request's block table
    points at, and the SAME layer's attention reads them -- so the result is right only
    if every layer's compute waits for its own fetch (H3).  Lengths log-uniform[128, 16k]
    (SURVEY.md §8(d) C5), reduced to 12 requests x 3 layers."""
    from paper_2510_13223_b200.kvstore import KVStore, ThreeStagePipeline
    shape = synth.Shape(3, 32, 8, 128)                        # Llama-3-8B head shape
    g = torch.Generator().manual_seed(5)
    lo, hi = np.log(128.0), np.log(16384.0)
    lens = np.exp(lo + (hi - lo) * torch.rand(12, generator=g).numpy()).astype(np.int64)
    dense = synth.gen_dense(shape, lens, seed=5)
    ks = np.stack([np.zeros(len(lens)), lens], 1).astype(np.int32)
    res = synth.place_shards(dense, ks, seed=5, spare_blocks=4)[0]
    nb = res.pool.shape[1]
    # prefix blocks: the first floor(0.5 * nblk) blocks of every request
    prefix = []
    for b in range(len(lens)):
        nblk = synth.ceil_div(int(lens[b]), 16)
        prefix += [int(x) for x in res.block_tables[b, : nblk // 2]]
    store_np = np.full((3, len(prefix) + 3, 2, 8, 16, 128), synth.BF16_NAN, dtype=np.uint16)
    store_np[:, :len(prefix)] = res.pool[:, prefix]           # the store holds the prefixes
    dev_np = res.pool.copy()
    dev_np[:, prefix] = synth.BF16_NAN                        # not resident yet on the GPU
    dev = bs.KVPool(3, nb, 8, 128)
    _fill(dev, dev_np)
    store = KVStore(3, store_np.shape[1], 8, 128)
    _fill(store.pool, store_np)
    q = torch.from_numpy(dense.q.view(np.int16)).view(torch.bfloat16).cuda()
    bt = torch.from_numpy(res.block_tables).cuda()
    ksd = torch.from_numpy(ks).cuda()
    B, sc = len(lens), synth.default_scale(128)
    o = torch.empty(3, B, 32, 128, device="cuda")
    m = torch.empty(3, B, 32, device="cuda")
    l = torch.empty(3, B, 32, device="cuda")
    ws = torch.zeros(max(16, bs.split_decode_attention_workspace_size(dev, B, 32, bt.shape[1])),
                     dtype=torch.uint8, device="cuda")

    def compute(layer):
        bs.split_decode_attention(dev, layer, q[layer], bt, ksd, 0, sc, o[layer], m[layer], l[layer], ws)

    pipe = ThreeStagePipeline(store, dev, 3, compute,
                              fetch_pairs=(list(range(len(prefix))), prefix), engine="ce")
    pipe.enqueue()
    torch.cuda.synchronize()
    for layer in range(3):
        ro, rm, rl = oracle.attention_shard(res.pool, layer, dense.q[layer], res.block_tables, ks, 0, sc)
        assert np.abs(o[layer].cpu().double().numpy() - ro).max() <= 5e-3
        assert np.abs((m[layer] + l[layer].log()).cpu().double().numpy() - (rm + np.log(rl))).max() <= 1e-4
