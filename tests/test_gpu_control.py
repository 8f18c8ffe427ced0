"""NEXT row F4 closed on the GPU (paper_2510_13223_b200/control.py): Alg. 1 planned with
Cost(m) from mechanism rates measured on this GPU (eq. 35) and its
moves executed by the F3 / F2 mechanisms (MigrateLayer / MigrateKVHeads, Alg. 1 lines
13 / 15).  Checks: the plan follows the measured costs (a rho between
the two modules' Benefit/Cost picks the cheaper one), every moved (layer, kv-head) unit is
bit-exact on its new device and untouched units keep the sentinel, moved weights are
equal, and attention over the new placement equals the oracle (north_star tolerances) and,
head range by head range, the same launch over the source pool bitwise (eq. 5)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

L, HKV, G, D = 4, 4, 2, 128
LENS = (1, 100, 333, 700)


@pytest.fixture(scope="module")
def bs():
    import paper_2510_13223_b200 as m
    m.lib()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def _setup(bs, weight_mib):
    from paper_2510_13223_b200.control import ModulePlacement
    shape = synth.Shape(L, HKV * G, HKV, D)
    dense = synth.gen_dense(shape, LENS, seed=21)
    ks = np.stack([np.zeros(len(LENS)), np.asarray(LENS)], 1).astype(np.int32)
    src = synth.place_shards(dense, ks, seed=22, spare_blocks=3)[0]
    nb = src.pool.shape[1]
    p0 = bs.KVPool(L, nb, HKV, D)
    p0.data.copy_(_dev(src.pool))
    nb1 = nb + 11
    p1 = bs.KVPool(L, nb1, HKV, D)
    p1.data.view(torch.int16).fill_(np.int16(np.uint16(synth.DST_SENTINEL).view(np.int16)))
    ids0 = sorted({int(x) for x in src.block_tables.ravel() if x >= 0})
    rng = np.random.default_rng(5)
    new = dict(zip(ids0, rng.permutation(nb1)[:len(ids0)].tolist()))   # device 1's placement
    bt1 = np.vectorize(lambda x: new.get(int(x), -1))(src.block_tables).astype(np.int32)
    i0 = torch.tensor(ids0, dtype=torch.int32, device="cuda")
    i1 = torch.tensor([new[x] for x in ids0], dtype=torch.int32, device="cuda")
    wn = weight_mib * 2**20 // 2
    g = torch.Generator(device="cuda").manual_seed(3)
    w0 = [torch.randn(wn, generator=g, device="cuda").to(torch.bfloat16) for _ in range(L)]
    w1 = [torch.zeros(wn, dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    pl = ModulePlacement([p0, p1], [i0, i1], [w0, w1])
    bts = [torch.from_numpy(src.block_tables).cuda(), torch.from_numpy(bt1).cuda()]
    return shape, dense, ks, src, pl, bts


def _costs(bs, pl, dense, ks, bts, shape):
    from paper_2510_13223_b200.control import MeasuredCosts
    scratch = bs.KVPool(L, pl.pools[0].num_blocks, HKV, D)   # same geometry as the source
    return MeasuredCosts.calibrate(pl.pools[0], scratch, pl.ids[0], pl.ids[0], pl.weights[0][0],
                                   _dev(dense.q[0]), bts[0], torch.from_numpy(ks).cuda(),
                                   synth.default_scale(D))


def _check_units(pl, moved):
    """moved: set of (layer, head) now on device 1; everything else still only on 0."""
    a, b = pl.pools[0].data, pl.pools[1].data
    i0, i1 = pl.ids[0].long(), pl.ids[1].long()
    sent = np.int16(np.uint16(synth.DST_SENTINEL).view(np.int16))
    for layer in range(L):
        for h in range(HKV):
            got = b[layer, i1, :, h].view(torch.int16)
            if (layer, h) in moved:
                assert torch.equal(got, a[layer, i0, :, h].view(torch.int16)), (layer, h)
            else:
                assert bool((got == int(sent)).all()), (layer, h)


def _check_attention(bs, pl, dense, ks, src, bts, shape):
    sc = synth.default_scale(D)
    B, hq = len(LENS), shape.hq
    ksd = torch.from_numpy(ks).cuda()
    for layer in range(L):
        q = _dev(dense.q[layer])
        o = torch.full((B, hq, D), float("nan"), device="cuda")
        m = torch.full((B, hq), float("nan"), device="cuda")
        l = torch.full((B, hq), float("nan"), device="cuda")
        pl.attention(layer, q, bts, ksd, sc, o, m, l)
        out = torch.empty(B, hq, D, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(B, hq, device="cuda")
        bs.merge_partials([o], [m], [l], out, lse)      # one part: bf16 conversion
        torch.cuda.synchronize()
        ref_o, ref_lse = oracle.attention_full([src.pool], [src.block_tables], layer, dense.q[layer],
                                               ks, sc)
        got = out.float().cpu().double().numpy()
        assert np.abs(got - ref_o).max() <= 2e-2
        assert (np.abs(got - ref_o).max(-1) / np.abs(ref_o).max(-1)).max() <= 1e-2
        assert np.abs(lse.cpu().double().numpy() - ref_lse).max() <= 1e-4
        # eq. 5: each head range moved to device 1 gives bitwise the same partial as the
        # same launch over the source pool
        for d, h0, nh in pl.head_runs(layer):
            if d == 0:
                continue
            o2, m2, l2 = (torch.full_like(x, float("nan")) for x in (o, m, l))
            wsn = bs.split_decode_attention_heads_workspace_size(pl.pools[0], B, nh, HKV, hq,
                                                                 bts[0].shape[1])
            ws = torch.zeros(max(16, wsn), dtype=torch.uint8, device="cuda")
            bs.split_decode_attention_heads(pl.pools[0], layer, h0, h0, nh, HKV, q, bts[0], ksd, 0, sc,
                                            o2, m2, l2, ws)
            torch.cuda.synchronize()
            rows = slice(h0 * G, (h0 + nh) * G)
            assert torch.equal(o[:, rows], o2[:, rows]) and torch.equal(m[:, rows], m2[:, rows])
            assert torch.equal(l[:, rows], l2[:, rows])


def test_measured_costs_drive_layer_moves(bs):
    from paper_2510_13223_b200.control import LAYER
    shape, dense, ks, src, pl, bts = _setup(bs, weight_mib=1)
    costs = _costs(bs, pl, dense, ks, bts, shape)
    assert min(costs.kv_layer_Bps, costs.kv_head_Bps, costs.weight_Bps) > 1e9 and costs.t_sync_s > 0
    assert [pl.load(d) for d in range(2)] == [2.0, 0.0]
    moves, load, n_layers, n_heads = pl.plan(costs, delta=0.3, rho=1.0)
    assert moves == [(LAYER, 0, 1), (LAYER, 0, 1)]       # 2.0/0.0 -> 1.5/0.5 -> 1.0/1.0
    assert load == [1.0, 1.0] and n_layers == [2, 2]
    pl.execute(moves)
    torch.cuda.synchronize()
    assert pl.executed == [("layer", 3, 0, 1), ("layer", 2, 0, 1)]
    assert [pl.load(d) for d in range(2)] == [1.0, 1.0]
    _check_units(pl, {(layer, h) for layer in (2, 3) for h in range(HKV)})
    for layer in range(L):
        same = torch.equal(pl.weights[1][layer], pl.weights[0][layer])
        assert same == (layer in (2, 3))
    _check_attention(bs, pl, dense, ks, src, bts, shape)
    # balanced: the next cycle plans nothing
    assert pl.plan(costs, delta=0.3, rho=1.0)[0] == []


def test_rho_between_measured_costs_picks_the_cheaper_module(bs):
    """Heavy layer weights make MigrateLayer's measured cost exceed MigrateKVHeads' (on an
    idle B200; the test follows whichever is cheaper as measured): with rho between the
    two Benefit/Cost ratios, Alg. 1 takes only the cheaper module (line 12 or line 14)."""
    from paper_2510_13223_b200.control import HEADS, LAYER
    shape, dense, ks, src, pl, bts = _setup(bs, weight_mib=512)
    costs = _costs(bs, pl, dense, ks, bts, shape)
    nblk = pl.ids[0].numel()
    page = pl.pools[0].chunk_bytes // (2 * HKV)
    c_layer = costs.layer_cost(nblk * pl.pools[0].chunk_bytes, 512 * 2**20)
    c_head = costs.head_cost(L * nblk * 2 * page)
    benefit = 2.0 - abs(1.5 - 0.5)                        # either module moves 0.5 of load
    rho = benefit / (c_layer * c_head) ** 0.5
    cheaper = HEADS if c_head < c_layer else LAYER
    assert pl.plan(costs, delta=0.3, rho=rho)[0] == [(cheaper, 0, 1)] * 2
    assert pl.plan(costs, delta=0.3, rho=benefit / min(c_layer, c_head) * 1.01)[0] == []


def test_kv_head_moves_executed(bs):
    """Layer migration unsupported on the overloaded device (Alg. 1 line 12 fails): the
    cycle moves KV heads (line 14) and MigrateKVHeads executes them."""
    from paper_2510_13223_b200.control import HEADS
    shape, dense, ks, src, pl, bts = _setup(bs, weight_mib=1)
    costs = _costs(bs, pl, dense, ks, bts, shape)
    moves, load, n_layers, n_heads = pl.plan(costs, delta=0.3, rho=1.0, supports_layer=[0, 1])
    assert moves == [(HEADS, 0, 1), (HEADS, 0, 1)] and load == [1.0, 1.0] and n_heads == [2, 2]
    pl.execute(moves)
    torch.cuda.synchronize()
    assert pl.executed == [("heads", 3, 0, 1), ("heads", 2, 0, 1)]
    assert pl.head_runs(0) == [(0, 0, 2), (1, 2, 2)]
    _check_units(pl, {(layer, h) for layer in range(L) for h in (2, 3)})
    assert all(not torch.equal(pl.weights[1][x], pl.weights[0][x]) for x in range(L))
    _check_attention(bs, pl, dense, ks, src, bts, shape)
